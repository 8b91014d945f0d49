#!/usr/bin/env bash
# round 2: ring_small DFS over neighbours in increasing edge cost, level cut at the first non-improving edge
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "config_plans or fuzz or sweep or search_configs or ga_search" > $O/r02aa_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/r02aa_pytest.txt
for i in 1 2; do timeout 300 python scripts/sweep_probe.py 4000000 >> $O/r02aa_sweep.jsonl 2>> $O/r02aa_sweep.err; done
for c in c4 c3 c2; do echo "$c" >> $O/r02aa_cfg.jsonl; timeout 300 python scripts/search_probe.py $c 10000 2 3 >> $O/r02aa_cfg.jsonl 2>&1; done
