# device vs host generation of GA init candidates (diagnostics)
mkdir -p gpurun_out
for m in 1000000 32; do
  HPG_DEVICE_GEN_MIN=$m timeout 900 python scripts/probe_perf.py c2,c3,c4 10000,100000 > gpurun_out/gen_$m.log 2>&1
done
