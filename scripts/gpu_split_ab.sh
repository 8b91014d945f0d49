# throughput-mode split swap waves: default vs off (diagnostics)
mkdir -p gpurun_out
timeout 300 python scripts/probe_perf.py c1,c2,c3,c4 10000 > gpurun_out/split_on.log 2>&1
HPG_GA_SPLIT_RUNS=1000000 timeout 300 python scripts/probe_perf.py c1,c2,c3,c4 10000 > gpurun_out/split_off.log 2>&1
