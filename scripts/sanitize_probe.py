"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck):
a device-GA search (c1, B=300), a host-GA search, a batched evaluation and a
sweep, all parity-checked against the committed goldens where one exists."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from golden_util import load, plan_from_golden  # noqa: E402
from paper_2512_12476_b200 import (CostModelConfig, Engine, SearchKnobs, load_topology,  # noqa: E402
                                   load_workflow, parse_topology, parse_workflow)

g = load("search_c1_b1000.json")
with Engine(parse_workflow(g["workflow"]), parse_topology(g["topology"])) as e:
    k = SearchKnobs.from_json(g["knobs"])
    k.budget = 300
    r = e.nested_sha_search(k)
    print("device-GA search consumed", r.consumed)
    ev = load("evalplans_c2.json")
with Engine(parse_workflow(ev["workflow"]), parse_topology(ev["topology"])) as e:
    plans = [plan_from_golden(x["plan"]) for x in ev["records"][:8]]
    out = e.evaluate(plans, CostModelConfig())
    print("evaluate", len(out))
with Engine(load_workflow(f"{ROOT}/fixtures/c4.workflow.json"),
            load_topology(f"{ROOT}/fixtures/c4.topology.json")) as e:
    st = e.sweep_resident(42, 0, 3000)
    print("sweep", st["n_feasible"], st["best_k"])
