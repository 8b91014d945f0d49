mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/chk_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/chk_tests.log
for i in 1 2; do timeout 600 python bench.py --no-cpu-baseline --no-sweep > gpurun_out/chk_bench$i.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/chk_bench$i.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel_share_of_step'], d['clocks'])"; done
