mkdir -p gpurun_out
for c in ${CFGS:-c2}; do
rm -f gpurun_out/galog_$c.txt
HPG_GA_LOG=gpurun_out/galog_$c.txt timeout 300 python scripts/probe_perf.py $c 10000 > gpurun_out/galog_probe_$c.log 2>&1
cat gpurun_out/galog_probe_$c.log | tail -2
done
