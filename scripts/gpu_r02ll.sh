#!/usr/bin/env bash
# round 2: TP ring bounds with the row's edges loaded up front (+ unrolled PP
# pair loop): parity, same-box A/B against the validated build
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > $O/r02ll_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/r02ll_pytest.txt
for pass in 1 2; do
  for v in base new; do
    if [ $v = base ]; then L=build/ab/libhpg_base.so; else L=paper_2512_12476_b200/libhpg.so; fi
    for c in c4 c3 c2 c1; do echo "$pass $v $c" >> $O/r02ll_cfg.jsonl; HPG_LIBRARY=$L timeout 300 python scripts/search_probe.py $c 10000 2 3 >> $O/r02ll_cfg.jsonl 2>&1; done
    echo "$pass $v sweep" >> $O/r02ll_sweep.jsonl; HPG_LIBRARY=$L timeout 300 python scripts/sweep_probe.py 4000000 >> $O/r02ll_sweep.jsonl 2>> $O/r02ll_sweep.err
  done
done
