# device-GA worker team A/B (diagnostics): HPG_GA_TEAM = 0 (auto), 1 (one warp), 2 (warp pair), 4
mkdir -p gpurun_out
HPG_GA_TEAM=4 timeout 600 python -m pytest tests -x -q -m gpu -k "search or ga" 2>&1 | tail -15 > gpurun_out/gateam_tests4.log
for t in 0 1 2 4; do
  HPG_GA_TEAM=$t timeout 300 python scripts/probe_perf.py c1,c2,c3,c4 10000 > gpurun_out/gateam_$t.log 2>&1
done
