"""GPU parity: the CUDA path (libhpg.so through the C ABI) against golden
vectors produced by the compiled reference (oracle/_ref/ref_dump).

The bar is bit-identity: every FP64 cost component, every feasibility flag,
every balanced split/weight, and for searches the consumed budget, b_m, the
incumbent trace, every arm record, every halving event, the survivor set after
every halving round and the chosen plan. (north_star asks for 1e-9 relative;
the kernels are built -fmad=false and restate the reference's operation order,
so the tests demand exact bits.)
"""
import pytest

from golden_util import check_breakdown, hx, load, plan_from_golden, same

pytestmark = pytest.mark.gpu


def _engine(wf_obj, topo_obj):
    from paper_2512_12476_b200 import Engine, parse_topology, parse_workflow
    return Engine(parse_workflow(wf_obj), parse_topology(topo_obj), device=0)


def _check_plan_eq(got: dict, want: dict, ctx=""):
    bad = []
    if [list(g) for g in got["groups"]] != [list(g) for g in want["groups"]]:
        bad.append(f"{ctx} groups {got['groups']} != {want['groups']}")
    if list(got["counts"]) != list(want["counts"]):
        bad.append(f"{ctx} counts {got['counts']} != {want['counts']}")
    for tid, l in want["layouts"].items():
        g = got["layouts"][int(tid)]
        for k in ("dp", "pp", "tp", "stage_layers"):
            if g[k] != l[k]:
                bad.append(f"{ctx} task {tid} {k}: {g[k]} != {l[k]}")
        if len(g["weights"]) != len(l["weights"]) or not all(
                same(a, hx(b)) for a, b in zip(g["weights"], l["weights"])):
            bad.append(f"{ctx} task {tid} weights differ")
    for tid, devs in want["assignment"].items():
        if list(got["assignment"][int(tid)]) != list(devs):
            bad.append(f"{ctx} task {tid} assignment differs")
    return bad


def _check_records(eng, recs, cfg, with_eval):
    plans = [plan_from_golden(r["plan"]) for r in recs]
    bds = eng.end_to_end_cost(plans, cfg)
    feas, req = eng.check_memory(plans, cfg)
    bal_d = eng.balance_data(plans, cfg)
    bal_l = eng.balance_layers(plans, cfg)
    bad = []
    for i, r in enumerate(recs):
        bad += check_breakdown(bds[i], r["e2e"], f"plan {i}")
        viol = r["violations"]
        if feas[i] != (len(viol) == 0):
            bad.append(f"plan {i}: feasible {feas[i]} vs {len(viol)} violations")
        for d, required, cap in viol:
            if not same(req[i][d], hx(required)):
                bad.append(f"plan {i}: required bytes on device {d}")
        for lab, got, want in (("balance_data", bal_d[i], r["balance_data"]),
                               ("balance_layers", bal_l[i], r["balance_layers"])):
            bad += _check_plan_eq(got, want, f"plan {i} {lab}")
    if with_eval:
        from paper_2512_12476_b200 import CostModelConfig
        ev = eng.evaluate(plans, CostModelConfig())
        for i, r in enumerate(recs):
            bad += _check_plan_eq(ev[i], r["evaluate"]["plan"], f"plan {i} evaluate")
            if not same(ev[i]["_e2e"], hx(r["evaluate"]["bd"]["end_to_end_s"])):
                bad.append(f"plan {i} evaluate e2e {ev[i]['_e2e']!r}")
    return bad


def test_fuzz_instances_bit_exact():
    """acceptance-#1-style random instances (tiny models, random topologies,
    random CostModelConfig incl. dbs/override/memory-model variations,
    embeddings, task subsets, async mode)."""
    from paper_2512_12476_b200 import CostModelConfig
    g = load("fuzz_eval.json")
    bad = []
    for i, r in enumerate(g["records"]):
        with _engine(r["workflow"], r["topology"]) as eng:
            cfg = CostModelConfig.from_json(r["cfg"])
            bad += [f"rec {i}: {b}" for b in _check_records(eng, [r], cfg, False)]
    assert not bad, "\n".join(bad[:20])


@pytest.mark.parametrize("cfg_name", ["c1", "c2", "c3", "c4", "n256"])
def test_config_plans_bit_exact(cfg_name):
    """A.5 generator + testutil::random_plan plans on the survey configs:
    end_to_end_cost, check_memory, balance_data, balance_layers and the
    search's evaluate() chain."""
    from paper_2512_12476_b200 import CostModelConfig
    g = load(f"evalplans_{cfg_name}.json")
    with _engine(g["workflow"], g["topology"]) as eng:
        bad = _check_records(eng, g["records"], CostModelConfig.from_json(g["cfg"]), True)
    assert not bad, "\n".join(bad[:20])


def check_search(res, gold, ctx=""):
    bad = []
    if res.consumed != gold["consumed"]:
        bad.append(f"{ctx} consumed {res.consumed} != {gold['consumed']}")
    if res.b_m != gold["b_m"]:
        bad.append(f"{ctx} b_m {res.b_m} != {gold['b_m']}")
    want_trace = [(c, hx(v)) for c, v in gold["trace"]]
    if len(res.trace) != len(want_trace) or not all(
            a[0] == b[0] and same(a[1], b[1]) for a, b in zip(res.trace, want_trace)):
        bad.append(f"{ctx} trace differs: {res.trace[:5]} vs {want_trace[:5]}")
    if len(res.arms) != len(gold["arms"]):
        bad.append(f"{ctx} arm count {len(res.arms)} != {len(gold['arms'])}")
    else:
        for i, (a, b) in enumerate(zip(res.arms, gold["arms"])):
            if a[0] != b[0] or a[1] != b[1] or a[3] != b[3] or not same(a[2], hx(b[2])):
                bad.append(f"{ctx} arm {i}: {a} != {b}")
                break
    want_h = [(h[0], h[1], h[2], hx(h[3]), hx(h[4])) for h in gold["halvings"]]
    if len(res.halvings) != len(want_h) or not all(
            a[:3] == b[:3] and same(a[3], b[3]) and same(a[4], b[4])
            for a, b in zip(res.halvings, want_h)):
        bad.append(f"{ctx} halvings differ")
    if res.survivors != gold["survivors"]:
        bad.append(f"{ctx} survivor sets differ")
    if bool(res.plan) != bool(gold["has_plan"]):
        bad.append(f"{ctx} has_plan {bool(res.plan)} != {gold['has_plan']}")
    elif res.plan:
        bad += _check_plan_eq(res.plan, gold["plan"], f"{ctx} chosen plan")
        bad += check_breakdown(res.breakdown, gold["breakdown"], f"{ctx} breakdown")
        if not same(res.plan["estimated_cost_s"], hx(gold["plan"]["estimated_cost_s"])):
            bad.append(f"{ctx} estimated_cost_s")
        if res.plan["provenance"]["budget"] != gold["plan"]["provenance"]["budget"]:
            bad.append(f"{ctx} provenance budget")
    return bad


SEARCH_GOLDENS = ["search_c1_b1000.json", "search_c2_b1000.json", "search_c3_b1000.json",
                  "search_c4_b1000.json", "search_c1_b10000.json", "search_c2_b10000.json",
                  "search_c3_b10000.json", "search_c4_b10000.json", "search_n256_b1000.json"]


@pytest.mark.parametrize("name", SEARCH_GOLDENS)
def test_search_configs_identical(name):
    from paper_2512_12476_b200 import SearchKnobs
    g = load(name)
    assert g["replay_consistent"]
    with _engine(g["workflow"], g["topology"]) as eng:
        res = eng.nested_sha_search(SearchKnobs.from_json(g["knobs"]))
    bad = check_search(res, g, name)
    assert not bad, "\n".join(bad[:20])


def test_search_fuzz_identical():
    """60 tiny searches with random knobs (balancing on/off, population,
    locality bias, swap sample, gg cap, quantization, level-1 filter/cap,
    overrides)."""
    from paper_2512_12476_b200 import SearchKnobs
    g = load("searchfuzz.json")
    bad = []
    for i, r in enumerate(g["records"]):
        with _engine(r["workflow"], r["topology"]) as eng:
            res = eng.nested_sha_search(SearchKnobs.from_json(r["knobs"]))
        bad += check_search(res, r, f"search {i}")
    assert not bad, "\n".join(bad[:30])


@pytest.mark.parametrize("cfg_name", ["c1", "c2", "c3", "c4"])
def test_ga_search_identical(cfg_name):
    """ga_search on its own (search.hpp:127-135): twelve arms per config with
    slices 1-400 and random seeds, feasible and infeasible; evaluations used,
    best member plan (bit-exact weights, splits, assignment), its cost and
    breakdown."""
    from paper_2512_12476_b200 import SearchKnobs
    g = load(f"ga_{cfg_name}.json")
    knobs = SearchKnobs.from_json(g["knobs"])
    bad = []
    with _engine(g["workflow"], g["topology"]) as eng:
        for i, r in enumerate(g["records"]):
            res = eng.ga_search(r["groups"], r["counts"], r["slice"], int(r["seed"]), knobs)
            ctx = f"{cfg_name} arm {i}"
            if res.consumed != r["evals"]:
                bad.append(f"{ctx} evals {res.consumed} != {r['evals']}")
            if bool(res.plan) != bool(r["has_plan"]):
                bad.append(f"{ctx} has_plan {bool(res.plan)} != {r['has_plan']}")
                continue
            if not res.plan:
                continue
            bad += _check_plan_eq(res.plan, r["plan"], ctx)
            if not same(res.arms[0][2], hx(r["cost"])):
                bad.append(f"{ctx} cost {res.arms[0][2]} != {hx(r['cost'])}")
            bad += check_breakdown(res.breakdown, r["breakdown"], ctx)
    assert not bad, "\n".join(bad[:20])


def test_sweep_c4_bit_exact():
    """config-5 generator on the GPU reproduces the reference's costs bit for
    bit (plans regenerated on the CPU by ref_dump from the same counters)."""
    from paper_2512_12476_b200 import Engine, load_topology, load_workflow
    from golden_util import FIXTURES
    import os
    g = load("sweep_c4.json")
    wf = load_workflow(os.path.join(FIXTURES, "c4.workflow.json"))
    topo = load_topology(os.path.join(FIXTURES, "c4.topology.json"))
    with Engine(wf, topo) as eng:
        out = eng.sweep(g["seed"], g["k0"], g["count"])
    want = [hx(v) for v in g["costs"]]
    mism = [i for i, (a, b) in enumerate(zip(out["costs"], want)) if not same(a, b)]
    assert not mism, f"{len(mism)} cost mismatches, first k={mism[:5]}"
    assert out["feasible"] == [bool(x) for x in g["feasible"]]
    assert out["n_feasible"] == g["n_feasible"]
    if g["n_feasible"]:
        assert out["best_k"] == g["best_k"] and same(out["best_cost"], hx(g["best"]))


def test_exhaustive_identical():
    """exhaustive_search on the device vs the reference (acceptance #2's twenty
    instances, test_search.cpp's tiny cases, the cap guard and 40 random
    pools): explored count, estimate, chosen plan, cost bits and breakdown,
    or the identical InputError when the estimate exceeds the cap."""
    from paper_2512_12476_b200 import InputError, SearchKnobs
    g = load("exhaustive.json")
    bad = []
    for r in g["records"]:
        obj = dict(r["knobs"])
        obj["exhaustive_cap"] = r["exhaustive_cap"]
        knobs = SearchKnobs.from_json(obj)
        with _engine(r["workflow"], r["topology"]) as eng:
            est = eng.exhaustive_space_estimate(knobs)
            if not same(est, hx(r["estimate"])):
                bad.append(f"{r['name']}: estimate {est!r} != {hx(r['estimate'])!r}")
            if "error" in r:
                try:
                    eng.exhaustive_search(knobs)
                    bad.append(f"{r['name']}: expected InputError")
                except InputError as e:
                    if r["error"] not in str(e):
                        bad.append(f"{r['name']}: error {e} != {r['error']}")
                continue
            res = eng.exhaustive_search(knobs)
        if res.info["consumed"] != r["explored"]:
            bad.append(f"{r['name']}: explored {res.info['consumed']} != {r['explored']}")
        if bool(res.plan) != bool(r["has_plan"]):
            bad.append(f"{r['name']}: has_plan {bool(res.plan)}")
            continue
        if res.plan:
            bad += _check_plan_eq(res.plan, r["plan"], r["name"])
            bad += check_breakdown(res.breakdown, r["breakdown"], r["name"])
            if not same(res.breakdown["end_to_end_s"], hx(r["cost"])):
                bad.append(f"{r['name']}: cost {res.breakdown['end_to_end_s']!r}")
            if not same(res.plan["estimated_cost_s"], hx(r["plan"]["estimated_cost_s"])):
                bad.append(f"{r['name']}: estimated_cost_s")
            if res.plan["provenance"]["budget"] != r["plan"]["provenance"]["budget"]:
                bad.append(f"{r['name']}: provenance budget")
    assert not bad, "\n".join(bad[:30])


def test_mixed_problem_sizes_in_one_process():
    """contexts with different shared-memory footprints in one process (the
    dynamic-smem opt-in must count the kernel's static shared memory: c3 then
    c4 once failed with an invalid launch configuration)"""
    import os
    from paper_2512_12476_b200 import Engine, SearchKnobs, load_topology, load_workflow
    from golden_util import FIXTURES
    for cfg in ("c3", "c4", "c1", "c4"):
        wf = load_workflow(os.path.join(FIXTURES, f"{cfg}.workflow.json"))
        topo = load_topology(os.path.join(FIXTURES, f"{cfg}.topology.json"))
        with Engine(wf, topo) as eng:
            res = eng.nested_sha_search(SearchKnobs(budget=2000, seed=42))
            assert res.consumed > 0 and res.plan is not None


@pytest.mark.parametrize("env", [{"HPG_DEVICE_GA": "0"},
                                 {"HPG_DEVICE_GA": "0", "HPG_DEVICE_GEN_MIN": "0"}],
                         ids=["host_ga", "host_ga_device_init"])
def test_host_ga_paths_identical(env):
    """The default search runs ga_run on the device (ga_kernel.cuh). The host
    coroutine GA in lockstep waves (HPG_DEVICE_GA=0), with init candidates
    made by the host pool or on the device (HPG_DEVICE_GEN_MIN=0), gives the
    same searches: c1/c2/n256 goldens, the 60 search fuzz cases and the
    ga_search arms, in a subprocess (the switches are read once)"""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-x",
                        os.path.join(here, "test_gpu_parity.py"), "-k",
                        "search_configs or search_fuzz or ga_search"],
                       env=dict(os.environ, **env), capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_sweep_stratified_sample_vs_reference():
    """config-5 parity at the benchmarked scale: the reference
    end_to_end_cost (oracle/_ref/ref_dump, run here on the host CPU) on a
    stratified 10^5-plan sample of the 10^8-plan sweep (100 blocks of 1000
    plans, block b at k = b * 10^6) against the GPU sweep of the same plans:
    every cost bit, every memory_feasible flag and the sample's argmin."""
    import os
    import struct
    import subprocess
    import tempfile
    from paper_2512_12476_b200 import Engine, load_topology, load_workflow
    from golden_util import FIXTURES
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = os.path.join(root, "oracle", "_ref", "ref_dump")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/ref_dump not built (needs /root/reference at build time)")
    wf_p = os.path.join(FIXTURES, "c4.workflow.json")
    tp_p = os.path.join(FIXTURES, "c4.topology.json")
    total, blocks, blen = 10 ** 8, 100, 1000
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "sample.bin")
        r = subprocess.run([exe, "sample_sweep", wf_p, tp_p, "42", str(total), str(blocks),
                            str(blen), str(max(1, len(os.sched_getaffinity(0)))), out],
                           capture_output=True, text=True, timeout=1200, check=True)
        raw = open(out, "rb").read()
    recs = [struct.unpack_from("<QQQ", raw, 24 * i) for i in range(blocks * blen)]
    stride = total // blocks
    bad, best = [], (float("inf"), None)
    with Engine(load_workflow(wf_p), load_topology(tp_p)) as eng:
        for b in range(blocks):
            got = eng.sweep(42, b * stride, blen)
            for i in range(blen):
                k, bits, feas = recs[b * blen + i]
                assert k == b * stride + i
                gbits = struct.unpack("<Q", struct.pack("<d", got["costs"][i]))[0]
                if gbits != bits or bool(feas) != got["feasible"][i]:
                    bad.append(k)
                if feas:
                    c = struct.unpack("<d", struct.pack("<Q", bits))[0]
                    if c < best[0]:
                        best = (c, k)
            if got["n_feasible"]:
                assert got["best_k"] >= b * stride and got["best_k"] < b * stride + blen
    assert not bad, f"{len(bad)} mismatches, first k={bad[:5]}"
    import json
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["best_k"] == best[1] and same(line["best_dec"], best[0])


def _search_golden_in_thread(name, device, out, key):
    from paper_2512_12476_b200 import Engine, SearchKnobs, parse_topology, parse_workflow
    try:
        g = load(name)
        with Engine(parse_workflow(g["workflow"]), parse_topology(g["topology"]),
                    device=device) as eng:
            for _ in range(2):
                res = eng.nested_sha_search(SearchKnobs.from_json(g["knobs"]))
                out.setdefault(key, []).extend(check_search(res, g, f"{name}@{device}"))
    except Exception as e:  # surfaced by the assertion below
        out.setdefault(key, []).append(repr(e))


def test_two_contexts_two_threads_one_device():
    """separate contexts are thread-safe (hpg.h): two threads drive two contexts
    on the same GPU at once (different problems, so different shared-memory
    sizes and launch parameters) and both reproduce the reference"""
    import threading
    out = {}
    ts = [threading.Thread(target=_search_golden_in_thread, args=(n, 0, out, n))
          for n in ("search_c1_b1000.json", "search_c2_b1000.json")]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    bad = [b for v in out.values() for b in v]
    assert len(out) == 2 and not bad, "\n".join(bad[:20])


def test_contexts_on_two_devices_one_process():
    """per-device launch state: contexts on GPU 0 and GPU 1 of one process, used
    from two threads, both reproduce the reference (needs >= 2 GPUs)"""
    import threading
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    out = {}
    ts = [threading.Thread(target=_search_golden_in_thread, args=(n, d, out, d))
          for d, n in ((0, "search_c2_b1000.json"), (1, "search_c1_b1000.json"))]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    bad = [b for v in out.values() for b in v]
    assert len(out) == 2 and not bad, "\n".join(bad[:20])
