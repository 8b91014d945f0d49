mkdir -p gpurun_out
for c in ${PCFGS:-c2 c4}; do
python scripts/prof_eval.py $c 8 > gpurun_out/pe_$c.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s 1 -c 1 -o gpurun_out/prof_$c \
  python scripts/prof_eval.py $c 8 > gpurun_out/ncu_$c.log 2>&1; echo "ncu $c rc=$?"
done
