#!/usr/bin/env bash
# round 2: c4 phase log with open-ring miss and DFS-edge counters
cd "$(dirname "$0")/.."
O=gpurun_out
rm -f $O/r02hh_galog_c4.txt
HPG_GA_LOG=$O/r02hh_galog_c4.txt timeout 300 python scripts/search_probe.py c4 10000 1 1 > $O/r02hh_probe.jsonl 2>&1
