# team-parallel init chunks: GA parity (auto and teams forced), then per-config timing and GA log
mkdir -p gpurun_out
timeout 600 python -m pytest tests -x -q -m gpu -k "search or ga" 2>&1 | tail -5 > gpurun_out/ti_tests.log
HPG_GA_TEAM=4 timeout 600 python -m pytest tests -x -q -m gpu -k "search or ga" 2>&1 | tail -5 >> gpurun_out/ti_tests.log
rm -f gpurun_out/galog_ti.txt
HPG_GA_LOG=gpurun_out/galog_ti.txt timeout 300 python scripts/c4_team_probe.py c1,c2,c3,c4 > gpurun_out/ti_probe_log.log 2>&1
timeout 300 python scripts/c4_team_probe.py c1,c2,c3,c4 > gpurun_out/ti_probe.log 2>&1
