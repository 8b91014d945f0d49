mkdir -p gpurun_out
python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -2 gpurun_out/bench.log
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-sweep > gpurun_out/b2.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-sweep > gpurun_out/ncu1.log 2>&1; echo "ncu1 rc=$?"
python scripts/probe_perf.py c2 1000 > gpurun_out/p.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:ga_kernel -s 20 -c 3 -o gpurun_out/prof_c2 \
  python scripts/probe_perf.py c2 1000 > gpurun_out/ncu2.log 2>&1; echo "ncu2 rc=$?"
[ -x oracle/_ref/shim_check ] && (timeout 600 oracle/_ref/shim_check > gpurun_out/shim.jsonl 2>gpurun_out/shim.err; echo "shim rc=$?"; tail -3 gpurun_out/shim.jsonl)
