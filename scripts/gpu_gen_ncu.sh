mkdir -p gpurun_out
HPG_DEVICE_GEN_MIN=0 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k search > gpurun_out/gen_parity.log 2>&1; echo parity rc=$?
HPG_DEVICE_GEN_MIN=32 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:gen_ga -c 200 --csv --log-file gpurun_out/gen_launches.csv python scripts/probe_perf.py c4 10000 > gpurun_out/gen_ncu.log 2>&1; echo ncu rc=$?
