"""Profiling driver: one eval_kernel launch in evaluate-chain mode over the
golden plans of a config (repeated to `reps` copies), preceded by a warm-up
launch. Run plain first, then under ncu with -s 1 -c 1."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from golden_util import load, plan_from_golden  # noqa: E402
from paper_2512_12476_b200 import CostModelConfig, Engine, parse_topology, parse_workflow  # noqa

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
g = load(f"evalplans_{cfg}.json")
eng = Engine(parse_workflow(g["workflow"]), parse_topology(g["topology"]))
plans = [plan_from_golden(r["plan"]) for r in g["records"]] * reps
eng.evaluate(plans, CostModelConfig())
eng.evaluate(plans, CostModelConfig())
print("ok", cfg, len(plans))
