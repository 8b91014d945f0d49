# larger budgets (SURVEY.md §8 D1 GPU-only B = 1e5, 1e6) on c2 and c4
mkdir -p gpurun_out
timeout 1500 python scripts/probe_perf.py ${CFGS:-c2,c4} ${BUDGETS:-100000,1000000} > gpurun_out/bigB.log 2>&1; echo rc=$?
