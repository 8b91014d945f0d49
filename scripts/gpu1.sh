nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -60 > gpurun_out/t1.log
cat gpurun_out/t1.log
