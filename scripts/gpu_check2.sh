mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/chk2_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/chk2_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
CFGS="c2 c4" bash scripts/gpu_galog.sh
timeout 600 python bench.py --no-cpu-baseline --no-sweep > gpurun_out/chk2_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/chk2_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['clocks'])"
