#!/usr/bin/env bash
# round 2: PP pairs grouped per cell (A) and batched open TP rings (A+B):
# parity on A+B, same-box A/B of base / A / A+B (search configs, sweep), and
# the c4 phase log of A+B
cd "$(dirname "$0")/.."
O=gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > $O/r02gg_pytest.txt 2>&1; echo "pytest rc=$?" >> $O/r02gg_pytest.txt
for pass in 1 2; do
  for v in base A AB; do
    case $v in base) L=build/ab/libhpg_base.so;; A) L=build/ab/libhpg_A.so;; AB) L=paper_2512_12476_b200/libhpg.so;; esac
    for c in c4 c3 c2 c1; do echo "$pass $v $c" >> $O/r02gg_cfg.jsonl; HPG_LIBRARY=$L timeout 300 python scripts/search_probe.py $c 10000 2 3 >> $O/r02gg_cfg.jsonl 2>&1; done
    echo "$pass $v sweep" >> $O/r02gg_sweep.jsonl; HPG_LIBRARY=$L timeout 300 python scripts/sweep_probe.py 4000000 >> $O/r02gg_sweep.jsonl 2>> $O/r02gg_sweep.err
  done
done
rm -f $O/r02gg_galog_c4.txt
HPG_GA_LOG=$O/r02gg_galog_c4.txt timeout 300 python scripts/search_probe.py c4 10000 1 1 > $O/r02gg_probe.jsonl 2>&1
