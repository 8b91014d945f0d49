#!/usr/bin/env bash
# round 2: ring_small with nearest-neighbour upper bounds and warp-shared pruning
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > $O/r02l_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/r02l_pytest.txt
for i in 1 2; do timeout 300 python scripts/sweep_probe.py 4000000 >> $O/r02l_sweep.jsonl 2>> $O/r02l_sweep.err; done
HPG_GA_LOG=$O/r02l_galog_c4.txt timeout 300 python scripts/search_probe.py c4 10000 2 2 > $O/r02l_c4_probe.jsonl 2>&1
timeout 300 python scripts/search_probe.py c4 10000 2 5 > $O/r02l_c4_probe_nolog.jsonl 2>&1
for c in c1 c2 c3; do timeout 300 python scripts/search_probe.py $c 10000 2 3 >> $O/r02l_cfg_probe.jsonl 2>&1; done
