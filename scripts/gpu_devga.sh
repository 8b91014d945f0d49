# device GA (ga_kernel) parity + A/B against the host offspring loop (diagnostics)
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "search" 2>&1 | tail -15 > gpurun_out/devga_tests.log
cat gpurun_out/devga_tests.log
timeout 300 python scripts/probe_perf.py ${CFGS:-c1,c2,c3,c4} ${BUDGETS:-10000} > gpurun_out/devga_on.log 2>&1
HPG_DEVICE_GA=0 timeout 300 python scripts/probe_perf.py ${CFGS:-c1,c2,c3,c4} ${BUDGETS:-10000} > gpurun_out/devga_off.log 2>&1
tail -5 gpurun_out/devga_on.log
