# device-GA team size per SHA round (diagnostics): forced 1 / 2 / 4 and auto, per-launch GA logs
mkdir -p gpurun_out
for t in 1 2 4 0; do
  rm -f gpurun_out/galog_t$t.txt
  HPG_GA_TEAM=$t HPG_GA_LOG=gpurun_out/galog_t$t.txt timeout 300 python scripts/c4_team_probe.py c1,c2,c3,c4 > gpurun_out/c4team_$t.log 2>&1
done
