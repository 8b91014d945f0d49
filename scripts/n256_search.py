"""256-GPU fleet: search at B=2000 and a 10^5 sweep run end to end (smoke of
the engine's size limits; diagnostics)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2512_12476_b200 import Engine, SearchKnobs, load_topology, load_workflow  # noqa

eng = Engine(load_workflow(f"{ROOT}/fixtures/n256.workflow.json"),
             load_topology(f"{ROOT}/fixtures/n256.topology.json"))
for B in (2000, 10000):
    t = time.perf_counter()
    r = eng.nested_sha_search(SearchKnobs(budget=B, seed=42))
    print(json.dumps(dict(B=B, wall=time.perf_counter() - t, consumed=r.consumed,
                          best=r.breakdown["end_to_end_s"] if r.breakdown else None,
                          waves=r.info["waves"])))
