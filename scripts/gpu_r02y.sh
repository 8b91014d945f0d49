#!/usr/bin/env bash
# round 2: link-class matrix in shared memory for the GA's helper-warp teams (c4: 16 KB)
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "search or ga_search" > $O/r02y_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/r02y_pytest.txt
for v in 0 1; do
  for c in c4 c3 c2 c1; do
    echo "CLS=$v $c" >> $O/r02y_cfg.jsonl
    HPG_GA_CLS_TEAM=$v timeout 300 python scripts/search_probe.py $c 10000 2 3 >> $O/r02y_cfg.jsonl 2>&1
  done
done
