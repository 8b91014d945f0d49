"""Sweep throughput probe: hpg_sweep_resident over `count` plans of the c4
config-5 generator; prints one JSON line."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_12476_b200 import Engine, load_topology, load_workflow  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
k0 = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = sys.argv[3] if len(sys.argv) > 3 else "c4"
fx = os.path.join(ROOT, "fixtures")
with Engine(load_workflow(f"{fx}/{cfg}.workflow.json"), load_topology(f"{fx}/{cfg}.topology.json")) as e:
    e.sweep_resident(42, k0, 100_000)
    t0 = time.perf_counter()
    st = e.sweep_resident(42, k0, count)
    wall = time.perf_counter() - t0
st["plans_per_s"] = count / (st["total_ms"] / 1000.0)
st["wall_s"] = wall
st["env"] = {k: v for k, v in os.environ.items() if k.startswith("HPG_")}
print(json.dumps(st), flush=True)
