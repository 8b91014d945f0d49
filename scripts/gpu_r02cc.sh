#!/usr/bin/env bash
# round 2: exact ring-memo keys + per-search memo reset: parity and timing
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py -x -q > $O/r02cc_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/r02cc_pytest.txt
for c in c4 c3 c2 c1; do echo "$c" >> $O/r02cc_cfg.jsonl; timeout 300 python scripts/search_probe.py $c 10000 2 3 >> $O/r02cc_cfg.jsonl 2>&1; done
timeout 300 python scripts/sweep_probe.py 4000000 >> $O/r02cc_sweep.jsonl 2>> $O/r02cc_sweep.err
