"""Benchmark: candidate plans evaluated/sec of HetRL's nested-SHA plan search.

Headline workload (BASELINE.json configs[3], the largest search scenario, which
fits one GPU): c4 = PPO Qwen2.5-32B on 128 GPUs of 4 types across 4 regions,
full nested successive-halving search with the per-arm genetic search and load
balancing, budget B=10^4 evaluations, seed 42, default knobs
(proj/samples/knobs.json). One step = one complete search. value = evaluations
consumed / device-timed seconds (max over ranks); e2e = the same through the C
ABI with host inputs (problem re-parsed and re-staged from host memory, search,
chosen plan + breakdown + trace read back, every step).

Beside the headline: c1-c3 at the same budget ("configs"), and the config-5
sweep ("c5_sweep": 10^8 plans of the counter-based generator on c4, sharded in
contiguous plan-index ranges across the ranks, with the reference's
end_to_end_cost timed on a stratified 10^5-plan sample on all host cores).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl engine|reference]
                  [--config c1..c4] [--budget B] [--sweep-plans P]

--impl reference times the unmodified reference planner (compiled from
/root/reference into oracle/_ref by oracle/Makefile) on the host CPU. The
reference search is single-threaded, so every search runs on one core; the K
timed searches run concurrently, one per physical core (pinned), and the value
is consumed / wall summed over searches, i.e. the one-core search rate.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "candidate plans evaluated/sec (nested SHA search incl. balancing)"
UNIT = "plans/s"
REF_DUMP = os.path.join(ROOT, "oracle", "_ref", "ref_dump")

# SURVEY.md Appendix A
CONFIGS = {
    "c1": "PPO Qwen-4B (proj/samples/workflow-ppo-4b.json) on 4xA100+4xL40S "
          "(generate_scenario 1, seed 7)",
    "c2": "GRPO Qwen2.5-7B on 16xA100+16xL40S (generate_scenario 1, seed 7)",
    "c3": "PPO Qwen2.5-14B on 64 GPUs of 3 types in 3 regions (generate_scenario 2, seed 7)",
    "c4": "PPO Qwen2.5-32B on 128 GPUs of 4 types (A100/L40S/L4/H100) across 4 regions",
}
SWEEP_PLANS = 10 ** 8
SWEEP_SAMPLE = (100, 1000)  # stratified CPU sample: 100 blocks x 1000 plans


def knobs_obj(budget, seed):
    # proj/samples/knobs.json with the bench budget / seed
    return dict(budget=budget, seed=seed, population=16, locality_bias=0.8,
                quantize_gpu_counts=1, level1_filter="off", gg_arm_cap=64, swap_pair_sample=8,
                balance_data=True, balance_layers=True, balance_seqlen=True, recompute=True)


def fixture(cfg):
    return (os.path.join(ROOT, "fixtures", f"{cfg}.workflow.json"),
            os.path.join(ROOT, "fixtures", f"{cfg}.topology.json"))


def config_obj(cfg, budget, seed, world):
    return {"workload": f"{cfg}: nested SHA search, {CONFIGS[cfg]}, B={budget}, seed {seed}, "
                        f"knobs=proj/samples/knobs.json",
            "budget": budget, "seed": seed, "parallelism": f"arms sharded x{world}",
            "l2": "flushed between steps (256 MiB device memset)"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "samples": len(sm),
                "reasons": sorted(reasons)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(key):
    """dram read+write bytes per launch from the committed ncu summary, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            return json.load(f)["kernels"][key]["dram_bytes_per_launch"]
    except Exception:
        return None


def cpu_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return model, os.cpu_count()


def physical_cores():
    """one logical CPU per physical core among the CPUs this process may use"""
    allowed = sorted(os.sched_getaffinity(0))
    seen, out = set(), []
    for c in allowed:
        base = f"/sys/devices/system/cpu/cpu{c}/topology"
        try:
            with open(f"{base}/core_id") as f:
                core = f.read().strip()
            with open(f"{base}/physical_package_id") as f:
                pkg = f.read().strip()
        except OSError:
            core, pkg = str(c), "0"
        if (pkg, core) not in seen:
            seen.add((pkg, core))
            out.append(c)
    return out


def _pin(cpu):
    return lambda: os.sched_setaffinity(0, {cpu})


def cpu_searches(cfg, budget, seed, count, cores, timeout=1500):
    """`count` reference searches of (cfg, budget, seed), run concurrently, at most
    one per physical core (each pinned to its core). Returns the parsed lines."""
    wf, tp = fixture(cfg)
    out, pending = [], list(range(count))
    while pending:
        wave = pending[:len(cores)]
        pending = pending[len(cores):]
        procs = [subprocess.Popen([REF_DUMP, "time_search", wf, tp, str(budget), str(seed)],
                                  stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True,
                                  preexec_fn=_pin(cores[i])) for i in range(len(wave))]
        for p in procs:
            o, e = p.communicate(timeout=timeout)
            if p.returncode != 0:
                raise RuntimeError(f"ref_dump time_search failed: {e[-500:]}")
            out.append(json.loads(o.strip().splitlines()[-1]))
    return out


def cpu_sample_sweep(threads, total=SWEEP_PLANS, seed=42, timeout=900):
    wf, tp = fixture("c4")
    blocks, blen = SWEEP_SAMPLE
    o = subprocess.run([REF_DUMP, "sample_sweep", wf, tp, str(seed), str(total), str(blocks),
                        str(blen), str(threads)],
                       capture_output=True, text=True, timeout=timeout, check=True)
    return json.loads(o.stdout.strip().splitlines()[-1])


# ---------------------------------------------------------------- reference arm

def run_reference(args, world, rank):
    if rank != 0:
        return
    if not os.path.exists(REF_DUMP):
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/ref_dump not built (needs /root/reference at build time)"}))
        return
    cores = physical_cores()
    model, ncpu = cpu_info()
    # warm-up: short searches of the same config (page cache, CPU frequency)
    cpu_searches(args.config, min(args.budget, 1000), args.seed, args.warmup, cores)
    rs = cpu_searches(args.config, args.budget, args.seed, args.steps, cores)
    consumed = sum(r["consumed"] for r in rs)
    wall = sum(r["wall_s"] for r in rs)
    value = consumed / wall
    conc = min(len(cores), args.steps)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * wall / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_obj(args.config, args.budget, args.seed, 1),
        "time_to_best_s": statistics.median(r["time_to_best_est_s"] for r in rs),
        "best_cost_s": rs[-1]["best_dec"],
        "consumed_per_step": rs[-1]["consumed"],
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "reference",
                         "sample": f"{args.steps} x nested_sha_search({args.config}, "
                                   f"B={args.budget}, seed {args.seed}), each single-threaded "
                                   f"on its own pinned physical core, {conc} at a time "
                                   f"({len(cores)} physical of {ncpu} logical CPUs, {model}); "
                                   f"value = sum(consumed) / sum(per-search wall)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------- engine arm

def run_engine(args, world, rank, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2512_12476_b200 import Engine, SearchKnobs, distutil, load_topology, load_workflow
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        return x if world == 1 else distutil.max_over_ranks(x)

    nid_cache = {}

    def search(eng, knobs):
        if world == 1:
            return eng.nested_sha_search(knobs)
        if id(eng) not in nid_cache:
            nid_cache[id(eng)] = distutil.broadcast_bytes(
                eng.nccl_unique_id() if rank == 0 else None, 0)
        return eng.nested_sha_search_dist(knobs, rank, world, nid_cache[id(eng)])

    def timed_searches(eng, knobs, steps):
        ms, infos, results = [], [], []
        for _ in range(steps):
            flush.zero_()
            barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            res = search(eng, knobs)
            e1.record()
            torch.cuda.synchronize()
            ms.append(max_over_ranks(e0.elapsed_time(e1)))
            infos.append(res.info)
            results.append(res)
        return ms, infos, results

    wf_path, tp_path = fixture(args.config)
    knobs = SearchKnobs.from_json(knobs_obj(args.budget, args.seed))
    eng = Engine(load_workflow(wf_path), load_topology(tp_path), device=local_rank)
    for _ in range(args.warmup):
        search(eng, knobs)
    # ---- device-resident timing (problem staged in HBM before the timed region) ----
    sampler = ClockSampler(local_rank)
    sampler.start()
    step_ms, infos, results = timed_searches(eng, knobs, args.steps)
    clocks = sampler.stop()
    # ---- end to end through the C ABI with host inputs: every step re-parses
    # the workflow/topology files, re-stages the problem from host memory
    # (hpg_restage), searches, and reads the chosen plan + breakdown + trace
    # back; the context (streams, buffers, NCCL communicator) persists like a
    # user's would ----
    e2e_ms, h2d, d2h = [], [], []
    for _ in range(args.steps):
        flush.zero_()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        wf2, topo2 = load_workflow(wf_path), load_topology(tp_path)
        eng.restage(wf2, topo2)
        r2 = search(eng, knobs)
        _ = (r2.plan, r2.breakdown, r2.trace)
        e1.record()
        torch.cuda.synchronize()
        e2e_ms.append(max_over_ranks(e0.elapsed_time(e1)))
        n = topo2.n
        prob_bytes = 8 * (3 * n) + n * n + 16 * 64
        h2d.append(r2.info["h2d_bytes"] + prob_bytes)
        d2h.append(r2.info["d2h_bytes"])
    eng.close()

    consumed = sum(i["consumed"] for i in infos)
    total_ms = sum(step_ms)
    value = consumed / (total_ms / 1000.0)
    e2e_value = consumed / (sum(e2e_ms) / 1000.0)
    # roofline of the dominant kernel, ga_kernel (the device GA of a SHA round:
    # its warps score every candidate): SURVEY.md §8 D1 canonical bytes of the
    # plans it scored / its CUDA-event time on the engine's stream
    eval_ms = sum(i["eval_kernel_ms"] for i in infos)
    eval_launches = sum(i["eval_launches"] for i in infos)
    cbytes = sum(i["canonical_bytes"] for i in infos)
    peak, peak_kind = measured_peaks()
    achieved = (cbytes / eval_launches) / ((eval_ms / eval_launches) / 1000.0) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (fixtures/ from the reference's generate_scenario and the "
                "4-type/4-region fleet of SURVEY.md App. A.4; no datasets)",
        "config": config_obj(args.config, args.budget, args.seed, world),
        "time_to_best_s": statistics.median(i["time_to_best_s"] for i in infos),
        "best_cost_s": results[-1].breakdown["end_to_end_s"] if results[-1].breakdown else None,
        "consumed_per_step": infos[-1]["consumed"],
        "e2e": {"value": e2e_value, "unit": UNIT,
                "h2d_bytes_per_step": int(statistics.median(h2d)),
                "d2h_bytes_per_step": int(statistics.median(d2h)),
                "ms_per_step": sum(e2e_ms) / args.steps},
        "roofline": {"bound": "hbm", "kernel": "ga_kernel", "achieved": achieved,
                     "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "peak_source": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)",
                     "traffic": ncu_traffic(f"ga_kernel_{args.config}"),
                     "algorithmic_bytes_per_launch": cbytes / eval_launches,
                     "avg_launch_ms": eval_ms / eval_launches,
                     "kernel_share_of_step": eval_ms / total_ms,
                     "note": "latency/issue-bound scalar FP64 gather work; HBM is not the "
                             "binding resource (SURVEY.md §8 D1)",
                     "traffic_note": "ncu --set full over every ga_kernel launch of one "
                                     "search of this config (profiles/ncu_summary.json), "
                                     "mean DRAM read+write bytes per launch"},
        "gpu_launches": sum(i["gpu_launches"] for i in infos),
        "waves_per_step": infos[-1]["waves"],
        "plans_scored_on_gpu_per_step": infos[-1]["plans_evaluated_gpu"],
        "clocks": clocks,
    }
    # the other search configs at the same budget (same timing rules, fewer steps)
    if not args.no_configs:
        extra = {}
        for cfg in ("c1", "c2", "c3", "c4"):
            if cfg == args.config:
                continue
            wf_p, tp_p = fixture(cfg)
            with Engine(load_workflow(wf_p), load_topology(tp_p), device=local_rank) as e:
                for _ in range(3):
                    search(e, knobs)
                ms, inf, res = timed_searches(e, knobs, 5)
                nid_cache.pop(id(e), None)
            extra[cfg] = {"plans_per_s": sum(i["consumed"] for i in inf) / (sum(ms) / 1000.0),
                          "ms_per_step": sum(ms) / len(ms), "consumed": inf[-1]["consumed"],
                          "time_to_best_s": statistics.median(i["time_to_best_s"] for i in inf),
                          "best_cost_s": res[-1].breakdown["end_to_end_s"]
                          if res[-1].breakdown else None,
                          "workload": config_obj(cfg, args.budget, args.seed, world)["workload"]}
        line["configs"] = extra
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args)
    if not args.no_sweep:
        line["c5_sweep"] = sweep_bench(args, world, rank)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def cpu_baseline(args):
    """bounded sample of the headline workload: one reference search of the
    same config at B=10^3 (about 10-20 s of one core)"""
    if not os.path.exists(REF_DUMP):
        return {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                "sample": "oracle/_ref/ref_dump not built"}
    model, ncpu = cpu_info()
    b = min(args.budget, 1000)
    r = cpu_searches(args.config, b, args.seed, 1, physical_cores())[0]
    return {"value": r["consumed"] / r["wall_s"], "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"1 x nested_sha_search({args.config}, B={b}, seed {args.seed}): "
                      f"{r['consumed']} evaluations in {r['wall_s']:.2f} s on 1 pinned core "
                      f"of {ncpu} ({model}); the reference is single-threaded",
            "time_to_best_est_s": r["time_to_best_est_s"]}


def sweep_bench(args, world, rank):
    """config-5 sweep on c4: 10^8 plans of the counter-based
    generator, scored with end_to_end_cost(CostModelConfig{}), argmin over the
    memory-feasible plans by (cost, k). The plan-index range is split into
    contiguous shards, one per rank (strong scaling: the total is fixed); the
    engine merges the (cost, k) argmin with one all-gather on its NCCL
    communicator (hpg_sweep_dist). Everything stays resident in HBM; only the
    reduction comes back."""
    import torch
    from paper_2512_12476_b200 import Engine, distutil, load_topology, load_workflow
    wf, tp = fixture("c4")
    total = args.sweep_plans
    k0, n = distutil.sweep_range(total, rank, world)
    with Engine(load_workflow(wf), load_topology(tp), device=torch.cuda.current_device()) as eng:
        nid = None
        if world > 1:
            nid = distutil.broadcast_bytes(eng.nccl_unique_id() if rank == 0 else None, 0)
        eng.sweep_resident(42, k0, 200000)  # warm-up (tables, allocations, code)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if world > 1:
            st = eng.sweep_dist(42, total, rank, world, nid)
        else:
            st = eng.sweep_resident(42, 0, total)
        wall_s = time.perf_counter() - t0
    total_ms = st["total_ms"] if world == 1 else 1000.0 * distutil.max_over_ranks(
        st["total_ms"] / 1000.0)
    peak, peak_kind = measured_peaks()
    # roofline of the dominant kernel (the fused generate + score kernel):
    # canonical bytes of the plans it scored / its CUDA-event time
    ach = st["canonical_bytes"] / (st["eval_ms"] / 1000.0) / 1e9
    out = {"plans": total, "n_gpus": world, "scaling": "strong",
           "plans_per_s": total / (total_ms / 1000.0), "total_ms": total_ms,
           "rank0_wall_ms": 1000.0 * wall_s, "kernel_ms_rank0": st["eval_ms"],
           "launches_rank0": st["launches"],
           "best_cost_s": st["best_cost"], "best_k": st["best_k"], "n_feasible": st["n_feasible"],
           "roofline": {"bound": "hbm", "kernel": "sweep_kernel", "achieved": ach, "peak": peak,
                        "unit": "GB/s", "frac": ach / peak,
                        "peak_source": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)",
                        "algorithmic_bytes_per_plan": st["canonical_bytes"] / max(1, n),
                        "traffic": ncu_traffic("sweep_kernel"),
                        "note": "rank 0's launches; canonical bytes per plan x plans / "
                                "kernel time"}}
    if rank == 0 and world == 1 and not args.no_cpu_baseline and os.path.exists(REF_DUMP):
        cores = physical_cores()
        r = cpu_sample_sweep(len(cores), total)
        model, ncpu = cpu_info()
        blocks, blen = SWEEP_SAMPLE
        out["cpu_baseline"] = {
            "value": r["plans_per_s"], "unit": "plans/s", "cores": r["threads"],
            "kind": "reference",
            "sample": f"reference end_to_end_cost on a stratified {r['count']}-plan sample of "
                      f"the same 10^8 (plan k = b*{r['stride']} + i, b < {blocks}, i < {blen}), "
                      f"{r['threads']} threads on {len(cores)} physical cores of {ncpu} "
                      f"({model}), {r['wall_s']:.2f} s",
            "extrapolated_full_sweep_s": total / r["plans_per_s"]}
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["engine", "reference"], default="engine")
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--budget", type=int, default=10000)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--sweep-plans", type=int, default=SWEEP_PLANS)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
    ap.add_argument("--no-configs", action="store_true")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_engine(args, world, rank, local_rank)


if __name__ == "__main__":
    main()
