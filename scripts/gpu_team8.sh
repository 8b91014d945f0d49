# device-GA team of eight (diagnostics): parity forced at 8, then 4 vs 8 per round
mkdir -p gpurun_out
HPG_GA_TEAM=8 timeout 600 python -m pytest tests -x -q -m gpu -k "search or ga" 2>&1 | tail -5 > gpurun_out/team8_tests.log
for t in 4 8; do
  rm -f gpurun_out/galog_t$t.txt
  HPG_GA_TEAM=$t HPG_GA_LOG=gpurun_out/galog_t$t.txt timeout 300 python scripts/c4_team_probe.py c1,c2,c3,c4 > gpurun_out/c4team_$t.log 2>&1
done
