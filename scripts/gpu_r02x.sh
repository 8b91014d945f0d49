#!/usr/bin/env bash
# round 2: exact rings by edge-cost thresholds (subset DP per lane) vs the DFS
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "config_plans or fuzz or sweep or search_configs or ga_search" > $O/r02x_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/r02x_pytest.txt
HPG_RING_DP_MIN=4 timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "config_plans or fuzz or sweep_c4 or search_configs" >> $O/r02x_pytest.txt 2>&1; echo "pytest dp4 rc=$?" >> $O/r02x_pytest.txt
for k in 9 7 6; do
  HPG_RING_DP_MIN=$k timeout 300 python scripts/sweep_probe.py 4000000 >> $O/r02x_sweep.jsonl 2>> $O/r02x_sweep.err
  for c in c4 c3; do
    echo "K=$k $c" >> $O/r02x_cfg.jsonl
    HPG_RING_DP_MIN=$k timeout 300 python scripts/search_probe.py $c 10000 2 3 >> $O/r02x_cfg.jsonl 2>&1
  done
done
