mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -30 > gpurun_out/t.log; cat gpurun_out/t.log
timeout 900 python scripts/probe_perf.py ${CFGS:-c1,c2,c3,c4} ${BUDGETS:-10000} ${SWEEP:-sweep} 2>&1 | tee gpurun_out/probe.log
