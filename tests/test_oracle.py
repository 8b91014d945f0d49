"""CPU: pin the C restatement oracle (oracle/hp_oracle.c) to the golden
vectors of the compiled reference, bit for bit. Runs without a GPU."""
import pytest

from golden_util import COMPONENTS, hx, load, same
from oracle_bind import Oracle


def _bd_bad(bd, gold, ids, ctx):
    bad = []
    for t, tid in enumerate(ids):
        want = gold["per_task"][str(tid)]
        for c in range(7):
            if not same(bd.per_task[t][c], hx(want[c])):
                bad.append(f"{ctx} task {tid} {COMPONENTS[c]} {bd.per_task[t][c]!r} != {hx(want[c])!r}")
    for k, v in (("reshard", "reshard_s"), ("sync", "sync_s"), ("e2e", "end_to_end_s")):
        if not same(getattr(bd, k), hx(gold[v])):
            bad.append(f"{ctx} {v}")
    if bool(bd.feasible) != bool(gold["memory_feasible"]):
        bad.append(f"{ctx} memory_feasible")
    return bad


def _layout_bad(o, pl, gold_plan, ctx):
    bad = []
    got = o.layouts_of(pl)
    for tid, l in gold_plan["layouts"].items():
        g = got[int(tid)]
        if g["stage_layers"] != l["stage_layers"]:
            bad.append(f"{ctx} task {tid} stage_layers {g['stage_layers']} != {l['stage_layers']}")
        if not all(same(a, hx(b)) for a, b in zip(g["weights"], l["weights"])):
            bad.append(f"{ctx} task {tid} weights")
    return bad


def _check(o, rec, cfg, with_eval):
    bad = []
    pl = o.plan(rec["plan"])
    bad += _bd_bad(o.e2e(pl, cfg), rec["e2e"], o.ids, "e2e")
    ok, req = o.check_memory(pl, cfg)
    if ok != (len(rec["violations"]) == 0):
        bad.append("check_memory verdict")
    for d, r, _ in rec["violations"]:
        if not same(req[d], hx(r)):
            bad.append(f"required bytes device {d}")
    pl = o.plan(rec["plan"])
    o.balance_data(pl, cfg)
    bad += _layout_bad(o, pl, rec["balance_data"], "balance_data")
    pl = o.plan(rec["plan"])
    o.balance_layers(pl, cfg)
    bad += _layout_bad(o, pl, rec["balance_layers"], "balance_layers")
    if with_eval:
        pl = o.plan(rec["plan"])
        bd = o.evaluate(pl, Oracle.cfg({}))
        bad += _bd_bad(bd, rec["evaluate"]["bd"], o.ids, "evaluate")
        bad += _layout_bad(o, pl, rec["evaluate"]["plan"], "evaluate")
    return bad


def test_oracle_fuzz_instances():
    g = load("fuzz_eval.json")
    bad = []
    for i, r in enumerate(g["records"]):
        o = Oracle(r["workflow"], r["topology"])
        bad += [f"rec {i}: {b}" for b in _check(o, r, Oracle.cfg(r["cfg"]), False)]
    assert not bad, "\n".join(bad[:20])


@pytest.mark.parametrize("cfg_name", ["c1", "c2", "c3", "c4"])
def test_oracle_config_plans(cfg_name):
    g = load(f"evalplans_{cfg_name}.json")
    o = Oracle(g["workflow"], g["topology"])
    recs = g["records"] if cfg_name in ("c1", "c2") else g["records"][:8]
    bad = []
    for i, r in enumerate(recs):
        bad += [f"plan {i}: {b}" for b in _check(o, r, Oracle.cfg(g["cfg"]), True)]
    assert not bad, "\n".join(bad[:20])


def test_oracle_reference_unit_pins():
    """known-answer values from the reference's unit tests
    (proj/tests/test_cost_model.cpp:46-61, :102-110)"""
    # pair_topology: 2 devices, 1 ms / 8 Gbps = 1e9 B/s
    topo = {"devices": [dict(id=f"dev-{i}", gpu_model="s", comp_tflops=1.0, mem_gb=1000.0,
                             hbm_gbps=1000.0, intra_node_gbps=600.0, node=f"n{i}", region="r0")
                        for i in range(2)],
            "region_links": [],
            "defaults": {"intra_region_latency_ms": 1.0, "intra_region_bandwidth_gbps": 8.0}}
    wf = {"algorithm": "ppo", "mode": "sync", "eta": 0.0,
          "batch": dict(global_batch=4, responses_per_prompt=1, seq_in=4, seq_out=2,
                        micro_batch_size=1),
          "tasks": [dict(id=6, kind=2, hidden_size=4, intermediate_size=8, num_layers=2,
                         include_embedding=False, vocab_size=0, precision_bytes=2)]}
    o = Oracle(wf, topo)
    import ctypes as C
    two = (C.c_int * 2)(0, 1)
    one = (C.c_int * 1)(0)
    assert o.L.hpo_ring(C.byref(o.p), one, 1, 12345.0) == 0.0
    assert abs(o.L.hpo_ring(C.byref(o.p), two, 2, 1e6) - 0.002) < 1e-15
    assert abs(o.L.hpo_ring(C.byref(o.p), two, 2, 320.0) - 0.00100032) < 1e-15
