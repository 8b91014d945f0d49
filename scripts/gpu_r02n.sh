#!/usr/bin/env bash
# round 2: ring variants A/B on one box: NN bound threshold K x NN step (shuffles / redux)
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "config_plans or fuzz or sweep_c4 or search_configs" > $O/r02n_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/r02n_pytest.txt
HPG_RING_REDUX=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "config_plans or fuzz or sweep_c4" >> $O/r02n_pytest.txt 2>&1; echo "pytest redux rc=$?" >> $O/r02n_pytest.txt
for rx in 0 1; do for k in 9 7; do
  HPG_RING_REDUX=$rx HPG_RING_NN_MIN=$k timeout 300 python scripts/sweep_probe.py 4000000 >> $O/r02n_sweep.jsonl 2>> $O/r02n_sweep.err
  for c in c4 c3; do
    echo "RX=$rx K=$k $c" >> $O/r02n_cfg.jsonl
    HPG_RING_REDUX=$rx HPG_RING_NN_MIN=$k timeout 300 python scripts/search_probe.py $c 10000 2 3 >> $O/r02n_cfg.jsonl 2>&1
  done
done; done
