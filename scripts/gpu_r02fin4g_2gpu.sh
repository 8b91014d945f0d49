#!/usr/bin/env bash
# round 2: 2-GPU parity (sharded search + sweep) and a 2-GPU bench line
cd "$(dirname "$0")/.."
O=gpurun_out
nvidia-smi -L > $O/r02fin4g_smi.txt 2>&1
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 \
  scripts/dist_check.py > $O/r02fin4g_dist_check.txt 2>&1; echo "rc=$?" >> $O/r02fin4g_dist_check.txt
timeout 1200 python -m pytest tests -m gpu -q -k "two_devices or multi_gpu" > $O/r02fin4g_pytest.txt 2>&1; echo "rc=$?" >> $O/r02fin4g_pytest.txt
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 \
  bench.py --gpus 2 --steps 5 --warmup 3 --no-configs > $O/r02fin4g_bench_n2.jsonl 2> $O/r02fin4g_bench_n2.err; echo "rc=$?" >> $O/r02fin4g_bench_n2.err
