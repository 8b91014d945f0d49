#!/usr/bin/env bash
# round 2: batched DP-ring bounds per stage
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "config_plans or fuzz or sweep_c4 or search_configs or ga_search" > $O/r02t_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/r02t_pytest.txt
for i in 1 2; do timeout 300 python scripts/sweep_probe.py 4000000 >> $O/r02t_sweep.jsonl 2>> $O/r02t_sweep.err; done
HPG_GA_LOG=$O/r02t_galog_c4.txt timeout 300 python scripts/search_probe.py c4 10000 2 2 > $O/r02t_c4_probe.jsonl 2>&1
for c in c4 c3; do echo "$c" >> $O/r02t_cfg.jsonl; timeout 300 python scripts/search_probe.py $c 10000 2 3 >> $O/r02t_cfg.jsonl 2>&1; done
