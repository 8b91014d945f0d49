# A/B of an alternative libhpg build (diagnostics): probe with the in-tree
# library, then with each build/var_*/libhpg.so (parity suite first).
mkdir -p gpurun_out
timeout 600 python scripts/probe_perf.py ${CFGS:-c1,c2,c3,c4} ${BUDGETS:-10000} > gpurun_out/ab_base.log 2>&1
cp paper_2512_12476_b200/libhpg.so /tmp/base.so
for v in build/var_*; do
  n=$(basename $v)
  cp $v/libhpg.so paper_2512_12476_b200/libhpg.so
  timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3 > gpurun_out/ab_${n}_tests.log
  timeout 600 python scripts/probe_perf.py ${CFGS:-c1,c2,c3,c4} ${BUDGETS:-10000} > gpurun_out/ab_${n}.log 2>&1
done
cp /tmp/base.so paper_2512_12476_b200/libhpg.so
timeout 600 python scripts/probe_perf.py ${CFGS:-c1,c2,c3,c4} ${BUDGETS:-10000} > gpurun_out/ab_base2.log 2>&1
