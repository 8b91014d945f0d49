#!/usr/bin/env bash
# round 2 final (batched open TP rings, PP lane groups): full GPU suite, smoke, bench + reference arm, launch list, ncu captures
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rs > $O/r02fin4_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/r02fin4_pytest.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/r02fin4_smoke.txt 2>&1; echo "smoke rc=$?" >> $O/r02fin4_smoke.txt
timeout 1200 python bench.py --steps 20 --warmup 5 > $O/r02fin4_bench.jsonl 2> $O/r02fin4_bench.err; echo "rc=$?" >> $O/r02fin4_bench.err
timeout 1700 python bench.py --impl reference --steps 20 --warmup 5 > $O/r02fin4_ref.jsonl 2> $O/r02fin4_ref.err; echo "rc=$?" >> $O/r02fin4_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02fin4_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-configs --no-cpu-baseline --sweep-plans 4000000 > $O/r02fin4_ncu_bench.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:ga_kernel --launch-skip 24 --launch-count 24 \
  -o /tmp/r02fin4_ga_c4 python scripts/search_probe.py c4 10000 1 1 > $O/r02fin4_ncu_ga.log 2>&1
ncu -i /tmp/r02fin4_ga_c4.ncu-rep --page raw --csv > $O/r02fin4_ga_c4_raw.csv 2>> $O/r02fin4_ncu_ga.log
timeout 600 ncu --set full --clock-control none -k regex:sweep_kernel -s 1 -c 1 \
  -o /tmp/r02fin4_sweep python scripts/sweep_probe.py 300000 > $O/r02fin4_ncu_sweep.log 2>&1
ncu -i /tmp/r02fin4_sweep.ncu-rep --page raw --csv > $O/r02fin4_sweep_raw.csv 2>> $O/r02fin4_ncu_sweep.log
