#!/usr/bin/env bash
# round 2: default re-check on the final build: class matrix in every GA
# worker's shared memory (HPG_GA_CLS_TEAM=2) and sweep CTA shapes
cd "$(dirname "$0")/.."
O=gpurun_out
for pass in 1 2; do
  for v in 1 2; do
    for c in c4 c3; do echo "$pass cls$v $c" >> $O/r02nn_cfg.jsonl; HPG_GA_CLS_TEAM=$v timeout 300 python scripts/search_probe.py $c 10000 2 3 >> $O/r02nn_cfg.jsonl 2>&1; done
  done
  for w in 8 16 81 4; do
    echo "$pass warps$w sweep" >> $O/r02nn_sweep.jsonl; HPG_SWEEP_WARPS=$w timeout 300 python scripts/sweep_probe.py 4000000 >> $O/r02nn_sweep.jsonl 2>> $O/r02nn_sweep.err
  done
done
