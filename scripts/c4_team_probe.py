"""Diagnostics: repeated searches per config (B = 10^4) to separate one-time from per-search costs."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_12476_b200 import Engine, SearchKnobs, load_topology, load_workflow  # noqa

KNOBS = dict(budget=10000, seed=42, population=16, locality_bias=0.8, quantize_gpu_counts=1,
             level1_filter="off", gg_arm_cap=64, swap_pair_sample=8, balance_data=True,
             balance_layers=True, balance_seqlen=True, recompute=True)
log = os.environ.get("HPG_GA_LOG")
for c in (sys.argv[1] if len(sys.argv) > 1 else "c4").split(","):
    e = Engine(load_workflow(f"{ROOT}/fixtures/{c}.workflow.json"),
               load_topology(f"{ROOT}/fixtures/{c}.topology.json"))
    for i in range(4):
        if log:
            with open(log, "a") as f:
                f.write(f"# {c} {i}\n")
        t0 = time.perf_counter()
        r = e.nested_sha_search(SearchKnobs.from_json(KNOBS))
        dt = time.perf_counter() - t0
        print(json.dumps(dict(cfg=c, i=i, wall_ms=1e3 * dt, eval_kernel_ms=r.info["eval_kernel_ms"],
                              batch_ms=r.info["batch_ms"])), flush=True)
    e.close()
