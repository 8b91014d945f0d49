mkdir -p gpurun_out
NG=${NG:-2}
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $NG --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus $NG --steps 5 --warmup 3 > gpurun_out/bench_n$NG.log 2>&1; echo rc=$?; tail -1 gpurun_out/bench_n$NG.log | cut -c1-900
