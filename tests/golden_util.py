"""Helpers for the golden fixtures under tests/golden/.

The fixtures are written by oracle/ref_dump (oracle/Makefile), which drives the
UNMODIFIED reference planner compiled from /root/reference/proj/src; every
double is a C99 hex float so comparisons are bit-exact. Regenerate with
tests/golden/regen.sh.
"""
import json
import os
import struct

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FIXTURES = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "fixtures")


def load(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def hx(v):
    return float.fromhex(v) if isinstance(v, str) else float(v)


def bits(x: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def same(a: float, b: float) -> bool:
    """bit-identical (NaN-safe)"""
    return bits(a) == bits(b)


def plan_from_golden(p):
    return dict(groups=p["groups"], counts=p["counts"],
                layouts={int(k): dict(dp=v["dp"], pp=v["pp"], tp=v["tp"],
                                      stage_layers=v["stage_layers"],
                                      weights=[hx(w) for w in v["weights"]])
                         for k, v in p["layouts"].items()},
                assignment={int(k): v for k, v in p["assignment"].items()})


COMPONENTS = ("comp", "tp", "pp", "dp", "bubble", "hbm", "total")


def check_breakdown(mine: dict, gold: dict, ctx=""):
    """Bit-exact CostBreakdown comparison; returns a list of mismatch strings."""
    bad = []
    for tid, vals in gold["per_task"].items():
        for c, v in zip(COMPONENTS, vals):
            got = mine["per_task"][int(tid)][c]
            if not same(got, hx(v)):
                bad.append(f"{ctx} task {tid} {c}: got {got!r} want {hx(v)!r}")
    for key in ("reshard_s", "sync_s", "end_to_end_s"):
        if not same(mine[key], hx(gold[key])):
            bad.append(f"{ctx} {key}: got {mine[key]!r} want {hx(gold[key])!r}")
    if bool(mine["memory_feasible"]) != bool(gold["memory_feasible"]):
        bad.append(f"{ctx} memory_feasible: got {mine['memory_feasible']} want "
                   f"{gold['memory_feasible']}")
    return bad
