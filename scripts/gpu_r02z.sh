#!/usr/bin/env bash
# round 2: link-class matrix in shared memory for every GA worker (2) vs teams only (1)
cd "$(dirname "$0")/.."
O=gpurun_out
HPG_GA_CLS_TEAM=2 timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "search_configs or ga_search" > $O/r02z_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/r02z_pytest.txt
for v in 1 2; do
  for c in c4 c1; do
    echo "CLS=$v $c" >> $O/r02z_cfg.jsonl
    HPG_GA_CLS_TEAM=$v timeout 300 python scripts/search_probe.py $c 10000 2 3 >> $O/r02z_cfg.jsonl 2>&1
  done
done
