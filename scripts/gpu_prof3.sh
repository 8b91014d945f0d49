mkdir -p gpurun_out
python scripts/probe_perf.py c2 10000 > gpurun_out/pl_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s 390 -c 3 -o gpurun_out/profl_c2 \
  python scripts/probe_perf.py c2 10000 > gpurun_out/ncul_c2.log 2>&1; echo "ncu c2 rc=$?"
python scripts/probe_perf.py c4 10000 > gpurun_out/pl_c4.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s 520 -c 3 -o gpurun_out/profl_c4 \
  python scripts/probe_perf.py c4 10000 > gpurun_out/ncul_c4.log 2>&1; echo "ncu c4 rc=$?"
