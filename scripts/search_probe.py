"""Search timeline probe: `warm` warm-up searches of a config, then `runs`
timed ones (wall + engine info); with HPG_GA_LOG set the engine appends its
per-SHA-round log. Used for the c4 critical-path analysis and under ncu."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_12476_b200 import Engine, SearchKnobs, load_topology, load_workflow  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
budget = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
warm = int(sys.argv[3]) if len(sys.argv) > 3 else 2
runs = int(sys.argv[4]) if len(sys.argv) > 4 else 3
K = dict(budget=budget, seed=42, population=16, locality_bias=0.8, quantize_gpu_counts=1,
         level1_filter="off", gg_arm_cap=64, swap_pair_sample=8, balance_data=True,
         balance_layers=True, balance_seqlen=True, recompute=True)
e = Engine(load_workflow(f"{ROOT}/fixtures/{cfg}.workflow.json"),
           load_topology(f"{ROOT}/fixtures/{cfg}.topology.json"))
k = SearchKnobs.from_json(K)
for _ in range(warm):
    e.nested_sha_search(k)
for _ in range(runs):
    t0 = time.perf_counter()
    r = e.nested_sha_search(k)
    w = time.perf_counter() - t0
    i = dict(r.info)
    i["wall_py_s"] = w
    i["best"] = r.breakdown["end_to_end_s"] if r.breakdown else None
    print(json.dumps({k2: i[k2] for k2 in ("consumed", "wall_s", "wall_py_s", "time_to_best_s",
                                             "gpu_launches", "eval_kernel_ms", "eval_launches",
                                             "host_ms", "batch_ms", "best")}), flush=True)
e.close()
