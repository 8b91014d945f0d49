mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node ${NG:-2} --master-addr 127.0.0.1 --master-port 29533 scripts/dist_check.py search_c1_b1000.json search_c2_b1000.json > gpurun_out/dist_devga.log 2>&1; echo "dist rc=$?"; tail -4 gpurun_out/dist_devga.log
NG=${NG:-2} bash scripts/gpu_scale.sh
