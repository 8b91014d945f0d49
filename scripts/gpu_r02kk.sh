#!/usr/bin/env bash
# round 2: one-warp GA workers with the evaluation carve in a global slab
# (more workers per SM in the wide rounds): parity, same-box A/B via
# HPG_GA_GCARVE=0/1, launch shapes
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > $O/r02kk_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/r02kk_pytest.txt
for pass in 1 2; do
  for v in 0 1; do
    for c in c4 c3 c2 c1; do echo "$pass gcarve$v $c" >> $O/r02kk_cfg.jsonl; HPG_GA_GCARVE=$v timeout 300 python scripts/search_probe.py $c 10000 2 3 >> $O/r02kk_cfg.jsonl 2>&1; done
  done
done
HPG_GA_LOG=$O/r02kk_galog_c4.txt timeout 300 python scripts/search_probe.py c4 10000 0 1 > $O/r02kk_probe.jsonl 2> $O/r02kk_smem.txt
