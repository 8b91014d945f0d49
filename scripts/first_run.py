"""First-search overhead in a fresh process (diagnostics)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_12476_b200 import Engine, SearchKnobs, load_topology, load_workflow  # noqa

cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
t0 = time.perf_counter()
eng = Engine(load_workflow(f"{ROOT}/fixtures/{cfg}.workflow.json"),
             load_topology(f"{ROOT}/fixtures/{cfg}.topology.json"))
t1 = time.perf_counter()
out = {"cfg": cfg, "create_s": t1 - t0}
for i in range(3):
    t = time.perf_counter()
    r = eng.nested_sha_search(SearchKnobs(budget=10000, seed=42))
    out[f"search{i}_s"] = time.perf_counter() - t
    out[f"batch{i}_ms"] = r.info["batch_ms"]
print(json.dumps(out))
