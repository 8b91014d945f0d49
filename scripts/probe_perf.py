"""Quick performance probe (not the bench): search wall time per config and
sweep throughput."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_12476_b200 import Engine, SearchKnobs, load_topology, load_workflow  # noqa

KNOBS = dict(budget=1000, seed=42, population=16, locality_bias=0.8, quantize_gpu_counts=1,
             level1_filter="off", gg_arm_cap=64, swap_pair_sample=8, balance_data=True,
             balance_layers=True, balance_seqlen=True, recompute=True)


def eng(c):
    return Engine(load_workflow(f"{ROOT}/fixtures/{c}.workflow.json"),
                  load_topology(f"{ROOT}/fixtures/{c}.topology.json"))


out = {}
cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["c1", "c2", "c3", "c4"]
budgets = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1000, 10000]
for c in cfgs:
    e = eng(c)
    e.nested_sha_search(SearchKnobs.from_json(dict(KNOBS, budget=2000)))  # warm-up
    for B in budgets:
        k = SearchKnobs.from_json(dict(KNOBS, budget=B))
        t0 = time.perf_counter()
        r = e.nested_sha_search(k)
        dt = time.perf_counter() - t0
        rec = dict(cfg=c, B=B, consumed=r.consumed, wall=dt, plans_s=r.consumed / dt,
                   best=r.breakdown["end_to_end_s"] if r.breakdown else None,
                   **{k_: r.info[k_] for k_ in ("waves", "gpu_launches", "plans_evaluated_gpu",
                                                "time_to_best_s", "eval_kernel_ms", "host_ms",
                                                "batch_ms")})
        print(json.dumps(rec), flush=True)
    e.close()
if "sweep" in sys.argv:
    e = eng("c4")
    e.sweep_resident(42, 0, 10000)
    for n in (100000, 1000000):
        t0 = time.perf_counter()
        st = e.sweep_resident(42, 0, n)
        dt = time.perf_counter() - t0
        print(json.dumps(dict(sweep=n, wall=dt, plans_s=n / dt, **st)), flush=True)
