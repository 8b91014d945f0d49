#!/usr/bin/env bash
# round 2: reference unit tests + acceptance on the engine; c4 search timeline; ncu of ga_kernel
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 900 oracle/_ref/unit_engine > $O/r02d_unit_engine.txt 2> $O/r02d_unit_engine.err; echo "rc=$?" >> $O/r02d_unit_engine.txt
timeout 1200 oracle/_ref/acceptance_engine > $O/r02d_acceptance_engine.txt 2> $O/r02d_acceptance_engine.err; echo "rc=$?" >> $O/r02d_acceptance_engine.txt
HPG_GA_LOG=$O/r02d_galog_c4.txt timeout 300 python scripts/search_probe.py c4 10000 2 3 > $O/r02d_c4_probe.jsonl 2>&1
timeout 300 python scripts/search_probe.py c4 10000 2 5 > $O/r02d_c4_probe_nolog.jsonl 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ga_kernel --launch-skip 30 --launch-count 40 \
  -o $O/r02d_ga_c4 python scripts/search_probe.py c4 10000 1 2 > $O/r02d_ncu.log 2>&1
