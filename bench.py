"""Benchmark: candidate plans evaluated/sec of HetRL's nested-SHA plan search.

Workload (BASELINE.json configs[1]): c2 = GRPO Qwen2.5-7B on 16xA100 +
16xL40S (reference generate_scenario(1, seed 7)), full nested successive-
halving search with the per-arm genetic search and load balancing, budget
B=10^4 evaluations, seed 42, default knobs (proj/samples/knobs.json). One
step = one complete search. value = evaluations consumed / device-timed
seconds (max over ranks); e2e = the same through the C ABI with host inputs
(context create/problem upload + search + result readout every step).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl engine|reference]

--impl reference times the unmodified reference planner (compiled from
/root/reference into oracle/_ref by oracle/Makefile) on the host CPU: the
reference search is single-threaded, so it runs on one core.
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


def knobs_obj(budget, seed):
    # proj/samples/knobs.json with the bench budget / seed
    return dict(budget=budget, seed=seed, population=16, locality_bias=0.8,
                quantize_gpu_counts=1, level1_filter="off", gg_arm_cap=64, swap_pair_sample=8,
                balance_data=True, balance_layers=True, balance_seqlen=True, recompute=True)


def fixture(cfg):
    return (os.path.join(ROOT, "fixtures", f"{cfg}.workflow.json"),
            os.path.join(ROOT, "fixtures", f"{cfg}.topology.json"))


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
        return 6650.0, "fallback"


def ncu_traffic(kernel):
    """dram read+write bytes per launch from the committed ncu summary, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            return json.load(f)["kernels"][kernel]["dram_bytes_per_launch"]
    except Exception:
        return None


def cpu_search(cfg, budget, seed, timeout=600):
    wf, tp = fixture(cfg)
    out = subprocess.run([REF_DUMP, "time_search", wf, tp, str(budget), str(seed)],
                         capture_output=True, text=True, timeout=timeout, check=True)
    return json.loads(out.stdout.strip().splitlines()[-1])


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


def run_reference(args, world, rank):
    if rank != 0:
        return
    if not os.path.exists(REF_DUMP):
        print(json.dumps({"impl": "reference", "unavailable":
                          "oracle/_ref/ref_dump not built (needs /root/reference at build time)"}))
        return
    for i in range(args.warmup):
        cpu_search(args.config, min(args.budget, 1000), args.seed + 1000 + i)
    consumed, wall, ttb = 0, 0.0, []
    best = None
    for i in range(args.steps):
        r = cpu_search(args.config, args.budget, args.seed)
        consumed += r["consumed"]
        wall += r["wall_s"]
        ttb.append(r["time_to_best_est_s"])
        best = r["best_dec"]
    value = consumed / wall
    model, ncpu = cpu_info()
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * wall / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_obj(args),
        "time_to_best_s": statistics.median(ttb), "best_cost_s": best,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "reference",
                         "sample": f"{args.steps} x nested_sha_search({args.config}, "
                                   f"B={args.budget}, seed {args.seed}) on 1 core of "
                                   f"{ncpu} ({model}); the reference is single-threaded"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_obj(args):
    return {"workload": f"{args.config}: nested SHA search, GRPO Qwen2.5-7B on 16xA100+16xL40S "
                        f"(scenario 1 seed 7), B={args.budget}, seed {args.seed}, "
                        f"knobs=proj/samples/knobs.json",
            "budget": args.budget, "seed": args.seed, "parallelism": f"arms sharded x{args.gpus}",
            "l2": "flushed between steps (256 MiB device memset)"}


def run_engine(args, world, rank, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2512_12476_b200 import Engine, SearchKnobs, load_topology, load_workflow
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    wf_path, tp_path = fixture(args.config)
    wf, topo = load_workflow(wf_path), load_topology(tp_path)
    knobs = SearchKnobs.from_json(knobs_obj(args.budget, args.seed))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    from paper_2512_12476_b200 import distutil

    def search(eng):
        if world == 1:
            return eng.nested_sha_search(knobs)
        nid = distutil.broadcast_bytes(eng.nccl_unique_id() if rank == 0 else None, 0)
        return eng.nested_sha_search_dist(knobs, rank, world, nid)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        return x if world == 1 else distutil.max_over_ranks(x)

    eng = Engine(wf, topo, device=local_rank)
    for _ in range(args.warmup):
        search(eng)
    # ---- device-resident timing (problem staged in HBM before the timed region) ----
    sampler = ClockSampler(local_rank)
    sampler.start()
    step_ms, infos, results = [], [], []
    for _ in range(args.steps):
        flush.zero_()
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        res = search(eng)
        e1.record()
        torch.cuda.synchronize()
        step_ms.append(max_over_ranks(e0.elapsed_time(e1)))
        infos.append(res.info)
        results.append(res)
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
        r2 = search(eng)
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
    # roofline of the dominant kernel: ga_kernel (the device GA of a SHA round,
    # whose warps evaluate every candidate; eval_kernel for the final
    # breakdown): canonical bytes of the plans evaluated / CUDA-event time
    eval_ms = sum(i["eval_kernel_ms"] for i in infos)
    eval_launches = sum(i["eval_launches"] for i in infos)
    cbytes = sum(i["canonical_bytes"] for i in infos)
    peak, peak_kind = measured_peaks()
    achieved = (cbytes / eval_launches) / ((eval_ms / eval_launches) / 1000.0) / 1e9
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (fixtures/ from the reference's generate_scenario; no datasets)",
        "config": config_obj(args),
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
                     "traffic": ncu_traffic("ga_kernel"),
                     "algorithmic_bytes_per_launch": cbytes / eval_launches,
                     "avg_launch_ms": eval_ms / eval_launches,
                     "kernel_share_of_step": eval_ms / total_ms,
                     "note": "latency/issue-bound scalar FP64 gather work; HBM is not the "
                             "binding resource (SURVEY.md §8 D1)",
                     "traffic_note": "ncu --set full replays a launch with flushed caches: "
                                     "its DRAM bytes are the kernel's SASS, the problem "
                                     "tables and the round's record pools, which stay in "
                                     "the 126 MB L2 while the round runs"},
        "gpu_launches": sum(i["gpu_launches"] for i in infos),
        "waves_per_step": infos[-1]["waves"],
        "plans_scored_on_gpu_per_step": infos[-1]["plans_evaluated_gpu"],
        "clocks": clocks,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args)
    if not args.no_sweep:
        line["c5_sweep"] = sweep_probe(args, world, rank)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def cpu_baseline(args):
    if not os.path.exists(REF_DUMP):
        return {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                "sample": "oracle/_ref/ref_dump not built"}
    model, ncpu = cpu_info()
    r = cpu_search(args.config, args.budget, args.seed)
    return {"value": r["consumed"] / r["wall_s"], "unit": UNIT, "cores": 1, "kind": "reference",
            "sample": f"1 x nested_sha_search({args.config}, B={args.budget}, seed {args.seed}), "
                      f"{r['wall_s']:.2f} s on 1 core of {ncpu} ({model})",
            "time_to_best_est_s": r["time_to_best_est_s"]}


def sweep_probe(args, world=1, rank=0):
    """config-5 sweep on c4: generator + e2e + argmin, all
    resident in HBM; reported beside the headline, not as it. With N GPUs the
    plan-index range is split into contiguous shards (weak scaling: each rank
    sweeps --sweep-plans plans) and the argmin merged with one all-gather."""
    import torch
    from paper_2512_12476_b200 import Engine, distutil, load_topology, load_workflow
    wf, tp = fixture("c4")
    total = args.sweep_plans * world
    k0, n = distutil.sweep_range(total, rank, world)
    with Engine(load_workflow(wf), load_topology(tp), device=torch.cuda.current_device()) as eng:
        eng.sweep_resident(42, k0, 20000)
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = eng.sweep_resident(42, k0, n)
        wall_s = time.perf_counter() - t0
    total_ms = st["total_ms"] if world == 1 else 1000.0 * distutil.max_over_ranks(
        st["total_ms"] / 1000.0)
    best_cost, best_k, n_feas = st["best_cost"], st["best_k"], st["n_feasible"]
    if world > 1:
        best_cost, best_k, n_feas = distutil.merge_argmin(best_cost, best_k, n_feas)
    peak, _ = measured_peaks()
    ach = st["canonical_bytes"] / (st["eval_ms"] / 1000.0) / 1e9
    return {"plans": total, "n_gpus": world, "scaling": "weak",
            "plans_per_s": total / (total_ms / 1000.0), "total_ms": total_ms,
            "rank0_wall_ms": 1000.0 * wall_s, "eval_ms_rank0": st["eval_ms"],
            "best_cost_s": best_cost, "best_k": best_k, "n_feasible": n_feas,
            "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                         "frac": ach / peak, "traffic": ncu_traffic("eval_kernel_sweep"),
                         "note": "rank 0's sweep kernels"}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["engine", "reference"], default="engine")
    ap.add_argument("--config", default="c2")
    ap.add_argument("--budget", type=int, default=10000)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--sweep-plans", type=int, default=1000000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sweep", action="store_true")
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
