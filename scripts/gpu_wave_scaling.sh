mkdir -p gpurun_out
for c in ${CFGS:-c2 c4}; do
  rm -f gpurun_out/wavescale_$c.txt
  HPG_BATCH_LOG=gpurun_out/wavescale_$c.txt timeout 600 python scripts/wave_scaling.py $c
  HPG_TEAM_POLICY=0 HPG_BATCH_LOG=gpurun_out/wavescale_${c}_t0.txt timeout 600 python scripts/wave_scaling.py $c
done
