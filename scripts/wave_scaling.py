"""Kernel time of one evaluate() wave vs wave size (diagnostics): the c2
golden plans replicated to n plans; HPG_BATCH_LOG must be set."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from golden_util import load, plan_from_golden  # noqa
from paper_2512_12476_b200 import CostModelConfig, Engine, parse_topology, parse_workflow  # noqa

cfg_name = sys.argv[1] if len(sys.argv) > 1 else "c2"
g = load(f"evalplans_{cfg_name}.json")
plans = [plan_from_golden(r["plan"]) for r in g["records"]]
cfg = CostModelConfig.from_json(g["cfg"])
log = os.environ["HPG_BATCH_LOG"]
with Engine(parse_workflow(g["workflow"]), parse_topology(g["topology"])) as eng:
    for mode in ("single", "mix"):
        for n in (1, 4, 16, 64, 148, 149, 222, 296, 444, 592, 888, 1184, 2368):
            ps = [plans[0]] * n if mode == "single" else [plans[i % len(plans)] for i in range(n)]
            for rep in range(4):
                open(log, "a").write(f"# {mode} {n} {rep}\n")
                eng.evaluate(ps, cfg)
