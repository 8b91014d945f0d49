#!/usr/bin/env bash
# round 2: full GPU suite, FP64 peak, compute-sanitizer
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rs > $O/r02e_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/r02e_pytest.txt
HPG_GA_LOG=$O/r02e_galog_c4.txt timeout 300 python scripts/search_probe.py c4 10000 2 2 > $O/r02e_c4_probe.jsonl 2>&1
timeout 120 scripts/fp64_peak > $O/r02e_fp64_peak.json 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_probe.py > $O/r02e_sanitizer_$tool.txt 2>&1
  echo "rc=$?" >> $O/r02e_sanitizer_$tool.txt
done
HPG_DEVICE_GA=0 timeout 1500 compute-sanitizer --tool memcheck --print-limit 50 python scripts/sanitize_probe.py > $O/r02e_sanitizer_memcheck_hostga.txt 2>&1
echo "rc=$?" >> $O/r02e_sanitizer_memcheck_hostga.txt
