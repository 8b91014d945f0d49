# ncu source-level capture of one ga_kernel launch (diagnostics)
mkdir -p gpurun_out
cat > /tmp/ga_one.py <<'PY'
import sys; sys.path.insert(0, '.')
from paper_2512_12476_b200 import Engine, SearchKnobs, load_topology, load_workflow
KNOBS = dict(budget=10000, seed=42, population=16, locality_bias=0.8, quantize_gpu_counts=1,
             level1_filter="off", gg_arm_cap=64, swap_pair_sample=8, balance_data=True,
             balance_layers=True, balance_seqlen=True, recompute=True)
e = Engine(load_workflow('fixtures/c2.workflow.json'), load_topology('fixtures/c2.topology.json'))
r = e.nested_sha_search(SearchKnobs.from_json(KNOBS))
print(r.consumed)
PY
timeout 900 ncu --set full --import-source on --clock-control none -k regex:ga_kernel -s ${SKIP:-14} -c 1 \
  -o gpurun_out/ga_c2 -f python /tmp/ga_one.py > gpurun_out/ga_ncu.log 2>&1
tail -3 gpurun_out/ga_ncu.log
