"""exhaustive_search timing probe: the reference (oracle/_ref/ref_dump, 1
core) vs the engine on the golden instance set (diagnostics, not the bench)."""
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2512_12476_b200 import Engine, InputError, SearchKnobs, parse_topology, parse_workflow  # noqa

with tempfile.TemporaryDirectory() as d:
    out = os.path.join(d, "exh.json")
    subprocess.run([os.path.join(ROOT, "oracle", "_ref", "ref_dump"), "exhaustive", "4242", "40",
                    out], check=True, env=dict(os.environ, HPG_REF_TIMING="1"),
                   capture_output=True)
    recs = json.load(open(out))["records"]
rows = []
for r in recs:
    if "error" in r or r["explored"] < 1000:
        continue
    obj = dict(r["knobs"])
    obj["exhaustive_cap"] = r["exhaustive_cap"]
    k = SearchKnobs.from_json(obj)
    with Engine(parse_workflow(r["workflow"]), parse_topology(r["topology"])) as eng:
        eng.exhaustive_search(k)  # warm-up
        t0 = time.perf_counter()
        res = eng.exhaustive_search(k)
        dt = time.perf_counter() - t0
    rows.append(dict(name=r["name"], explored=r["explored"], raw=res.info["budget"],
                     ref_s=r["ref_wall_s"], gpu_s=dt, speedup=r["ref_wall_s"] / dt,
                     same_cost=res.breakdown["end_to_end_s"] == float.fromhex(r["cost"])))
    print(json.dumps(rows[-1]), flush=True)
