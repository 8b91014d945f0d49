#!/usr/bin/env bash
# round 2: ring_small variants (nearest-neighbour bound from ring size K) on sweep / c3 / c4
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "config_plans or fuzz or sweep_c4" > $O/r02m_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/r02m_pytest.txt
for k in 9 8 7; do
  HPG_RING_NN_MIN=$k timeout 300 python scripts/sweep_probe.py 4000000 >> $O/r02m_sweep.jsonl 2>> $O/r02m_sweep.err
  for c in c4 c3; do
    echo "K=$k $c" >> $O/r02m_cfg.jsonl
    HPG_RING_NN_MIN=$k timeout 300 python scripts/search_probe.py $c 10000 2 3 >> $O/r02m_cfg.jsonl 2>&1
  done
done
