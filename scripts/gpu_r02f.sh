#!/usr/bin/env bash
# round 2: kernels with __grid_constant__ problem params (no local copies): parity + sweep + c4 search timing
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "sweep or search_configs or config_plans or fuzz or ga_search" > $O/r02f_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/r02f_pytest.txt
for cfg in "1 1 8" "1 2 8" "1 1 4" "0 0 8"; do
  set -- $cfg
  HPG_SWEEP_SORT=$1 HPG_SWEEP_SYNC=$2 HPG_SWEEP_WARPS=$3 timeout 300 python scripts/sweep_probe.py 2000000 >> $O/r02f_sweep.jsonl 2>> $O/r02f_sweep.err
done
HPG_GA_LOG=$O/r02f_galog_c4.txt timeout 300 python scripts/search_probe.py c4 10000 2 2 > $O/r02f_c4_probe.jsonl 2>&1
timeout 300 python scripts/search_probe.py c4 10000 2 5 > $O/r02f_c4_probe_nolog.jsonl 2>&1
HPG_SWEEP_SORT=1 HPG_SWEEP_SYNC=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:sweep_kernel -s 1 -c 1 \
  -o /tmp/r02f_sweep python scripts/sweep_probe.py 300000 > $O/r02f_ncu.log 2>&1
ncu -i /tmp/r02f_sweep.ncu-rep --page raw --csv > $O/r02f_sweep_raw.csv 2>> $O/r02f_ncu.log
