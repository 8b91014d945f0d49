#!/usr/bin/env bash
# round 2: GA worker shared-memory budget per team size (diagnostic)
cd "$(dirname "$0")/.."
O=gpurun_out
HPG_GA_LOG=/tmp/galog.txt timeout 300 python scripts/search_probe.py c4 10000 0 1 > $O/r02jj_probe.jsonl 2> $O/r02jj_smem.txt
HPG_GA_LOG=/tmp/galog2.txt timeout 300 python scripts/search_probe.py c2 10000 0 1 >> $O/r02jj_probe.jsonl 2>> $O/r02jj_smem.txt
