#!/usr/bin/env bash
# round 2: sweep_kernel parity + occupancy sweep + ncu of the sweep kernel
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sweep" > $O/r02b_pytest.txt 2>&1
echo "pytest rc=$?" >> $O/r02b_pytest.txt
for w in 8 4 2; do
  for slab in 0 16384 12288 8192; do
    HPG_SWEEP_WARPS=$w HPG_SWEEP_SLAB=$slab timeout 300 python scripts/sweep_probe.py 2000000 >> $O/r02b_probe.jsonl 2>> $O/r02b_probe.err
  done
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:sweep_kernel -s 1 -c 1 \
  -o $O/r02b_sweep python scripts/sweep_probe.py 300000 > $O/r02b_ncu.log 2>&1
echo "ncu rc=$?" >> $O/r02b_ncu.log
