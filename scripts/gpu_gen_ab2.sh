# repeated A/B: device generation threshold (diagnostics)
mkdir -p gpurun_out
for m in 1000000 32 1000000 32; do
  HPG_DEVICE_GEN_MIN=$m timeout 900 python scripts/probe_perf.py c3,c4 10000,10000,10000 >> gpurun_out/genab_$m.log 2>&1
done
