#!/usr/bin/env bash
# round 2: 4-GPU parity (sharded searches + sweep) and a 4-GPU bench line
cd "$(dirname "$0")/.."
O=gpurun_out
nvidia-smi -L > $O/r02fin4h_smi.txt 2>&1
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29551 \
  scripts/dist_check.py > $O/r02fin4h_dist_check.txt 2>&1; echo "rc=$?" >> $O/r02fin4h_dist_check.txt
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29552 \
  bench.py --gpus 4 --steps 5 --warmup 3 > $O/r02fin4h_bench_n4.jsonl 2> $O/r02fin4h_bench_n4.err; echo "rc=$?" >> $O/r02fin4h_bench_n4.err
