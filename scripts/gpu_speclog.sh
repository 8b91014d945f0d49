# speculation hit rate per lockstep round (diagnostics)
mkdir -p gpurun_out
for c in ${CFGS:-c2 c4}; do
HPG_SPEC_LOG=gpurun_out/spec_$c.txt timeout 600 python - <<PY
import sys; sys.path.insert(0, '.')
from paper_2512_12476_b200 import Engine, SearchKnobs, load_topology, load_workflow
KNOBS = dict(budget=10000, seed=42, population=16, locality_bias=0.8, quantize_gpu_counts=1,
             level1_filter="off", gg_arm_cap=64, swap_pair_sample=8, balance_data=True,
             balance_layers=True, balance_seqlen=True, recompute=True)
e = Engine(load_workflow('fixtures/$c.workflow.json'), load_topology('fixtures/$c.topology.json'))
r = e.nested_sha_search(SearchKnobs.from_json(KNOBS))
print('$c', r.consumed, r.info['waves'])
PY
done
