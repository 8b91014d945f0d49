mkdir -p gpurun_out
for c in ${PCFGS:-c2 c4}; do
python scripts/probe_perf.py $c 3000 > gpurun_out/p_$c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s ${SKIP:-60} -c ${CNT:-4} -o gpurun_out/prof_$c \
  python scripts/probe_perf.py $c 3000 > gpurun_out/ncu_$c.log 2>&1; echo "ncu $c rc=$?"
done
