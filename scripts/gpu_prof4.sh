# ncu full capture of a few mid-search eval_kernel launches (c2)
mkdir -p gpurun_out
python scripts/probe_perf.py c2 10000 > gpurun_out/p4_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s ${SKIP:-230} -c ${COUNT:-6} -o gpurun_out/prof4_c2 \
  python scripts/probe_perf.py c2 10000 > gpurun_out/ncu4_c2.log 2>&1; echo "ncu c2 rc=$?"
