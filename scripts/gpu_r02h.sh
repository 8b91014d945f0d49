#!/usr/bin/env bash
# round 2: parity after the host-side search changes, search timing, full bench + reference arm
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "search or ga_search or host_ga" > $O/r02h_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/r02h_pytest.txt
HPG_GA_LOG=$O/r02h_galog_c4.txt timeout 300 python scripts/search_probe.py c4 10000 2 2 > $O/r02h_c4_probe.jsonl 2>&1
timeout 1200 python bench.py --steps 20 --warmup 5 > $O/r02h_bench.jsonl 2> $O/r02h_bench.err; echo "rc=$?" >> $O/r02h_bench.err
timeout 1700 python bench.py --impl reference --steps 20 --warmup 5 > $O/r02h_ref.jsonl 2> $O/r02h_ref.err; echo "rc=$?" >> $O/r02h_ref.err
