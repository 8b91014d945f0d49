# team policy A/B (diagnostics): 0 = one warp per plan, 1 = teams in small waves, 2 = + pairs in medium waves
mkdir -p gpurun_out
for pol in 0 1 2; do
  HPG_TEAM_POLICY=$pol timeout 600 python scripts/probe_perf.py c1,c2,c3,c4 10000 sweep > gpurun_out/team_$pol.log 2>&1
done
