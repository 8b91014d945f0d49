#!/usr/bin/env bash
# round 2: where the c4 GA's evaluation time goes (HPG_GA_LOG phase counters)
cd "$(dirname "$0")/.."
O=gpurun_out
rm -f $O/r02ff_galog_c4.txt
HPG_GA_LOG=$O/r02ff_galog_c4.txt timeout 300 python scripts/search_probe.py c4 10000 1 1 > $O/r02ff_probe.jsonl 2>&1
