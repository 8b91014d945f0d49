#!/usr/bin/env bash
# round 2: source-level profile of the sweep kernel (instructions and stalls per SASS line)
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:sweep_kernel -s 1 -c 1 \
  -o /tmp/r02i_sweep python scripts/sweep_probe.py 300000 > $O/r02i_ncu.log 2>&1
ncu -i /tmp/r02i_sweep.ncu-rep --page source --csv --print-source sass > $O/r02i_sweep_source.csv 2>> $O/r02i_ncu.log
gzip -f $O/r02i_sweep_source.csv
ncu -i /tmp/r02i_sweep.ncu-rep --page raw --csv > $O/r02i_sweep_raw.csv 2>> $O/r02i_ncu.log
