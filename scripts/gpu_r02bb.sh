#!/usr/bin/env bash
# round 2: geometry memo after the memory gate (team stage job without geometry)
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "config_plans or fuzz or search or ga_search or exhaustive" > $O/r02bb_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/r02bb_pytest.txt
for c in c4 c3 c2 c1; do echo "$c" >> $O/r02bb_cfg.jsonl; timeout 300 python scripts/search_probe.py $c 10000 2 3 >> $O/r02bb_cfg.jsonl 2>&1; done
timeout 300 python scripts/sweep_probe.py 4000000 >> $O/r02bb_sweep.jsonl 2>> $O/r02bb_sweep.err
