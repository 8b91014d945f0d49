#!/usr/bin/env bash
# round 2: reference unit tests + acceptance on the engine; c4 search timeline;
# ncu of ga_kernel (summarised on the box: the .ncu-rep is too large to bring back)
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 900 oracle/_ref/unit_engine > $O/r02d_unit_engine.txt 2> $O/r02d_unit_engine.err; echo "rc=$?" >> $O/r02d_unit_engine.txt
timeout 1200 oracle/_ref/acceptance_engine > $O/r02d_acceptance_engine.txt 2> $O/r02d_acceptance_engine.err; echo "rc=$?" >> $O/r02d_acceptance_engine.txt
HPG_GA_LOG=$O/r02d_galog_c4.txt timeout 300 python scripts/search_probe.py c4 10000 2 3 > $O/r02d_c4_probe.jsonl 2>&1
timeout 300 python scripts/search_probe.py c4 10000 2 5 > $O/r02d_c4_probe_nolog.jsonl 2>&1
for s in 0 1; do
  HPG_SWEEP_SYNC=1 HPG_SWEEP_SORT=$s timeout 300 python scripts/sweep_probe.py 2000000 >> $O/r02d_sweep.jsonl 2>> $O/r02d_sweep.err
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ga_kernel --launch-skip 24 --launch-count 24 \
  -o /tmp/r02d_ga_c4 python scripts/search_probe.py c4 10000 1 1 > $O/r02d_ncu.log 2>&1
ncu -i /tmp/r02d_ga_c4.ncu-rep --page raw --csv > $O/r02d_ga_c4_raw.csv 2>> $O/r02d_ncu.log
ncu -i /tmp/r02d_ga_c4.ncu-rep --page source --csv --print-source sass > $O/r02d_ga_c4_source.csv 2>> $O/r02d_ncu.log
gzip -f $O/r02d_ga_c4_source.csv
