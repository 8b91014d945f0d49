#!/usr/bin/env bash
# round 2: sweep CTA shapes (warps x CTAs per SM): 8x2, 16x1, 8x1, 4x4
cd "$(dirname "$0")/.."
O=gpurun_out
for w in 16 81 8 4; do
  HPG_SWEEP_WARPS=$w timeout 300 python scripts/sweep_probe.py 4000000 >> $O/r02r_sweep.jsonl 2>> $O/r02r_sweep.err
done
HPG_SWEEP_WARPS=16 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sweep" > $O/r02r_pytest16.txt 2>&1; echo "rc=$?" >> $O/r02r_pytest16.txt
HPG_SWEEP_WARPS=81 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sweep" > $O/r02r_pytest81.txt 2>&1; echo "rc=$?" >> $O/r02r_pytest81.txt
