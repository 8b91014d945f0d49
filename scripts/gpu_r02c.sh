#!/usr/bin/env bash
# round 2: sweep_kernel phase barriers A/B (instruction-cache sharing)
cd "$(dirname "$0")/.."
O=gpurun_out
for sync in 0 1; do
  for w in 8 4; do
    HPG_SWEEP_SYNC=$sync HPG_SWEEP_WARPS=$w timeout 300 python scripts/sweep_probe.py 2000000 >> $O/r02c_probe.jsonl 2>> $O/r02c_probe.err
  done
done
HPG_SWEEP_SYNC=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sweep" > $O/r02c_pytest.txt 2>&1
HPG_SWEEP_SYNC=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:sweep_kernel -s 1 -c 1 \
  -o $O/r02c_sweep_sync python scripts/sweep_probe.py 300000 > $O/r02c_ncu.log 2>&1
