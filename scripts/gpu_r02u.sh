#!/usr/bin/env bash
# round 2: run-head-only staging of the device GA rounds: parity + c4 timing
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "search or ga_search or mixed" > $O/r02u_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/r02u_pytest.txt
HPG_GA_LOG=$O/r02u_galog_c4.txt timeout 300 python scripts/search_probe.py c4 10000 2 2 > $O/r02u_c4_probe.jsonl 2>&1
for c in c4 c2; do echo "$c" >> $O/r02u_cfg.jsonl; timeout 300 python scripts/search_probe.py $c 10000 2 3 >> $O/r02u_cfg.jsonl 2>&1; done
