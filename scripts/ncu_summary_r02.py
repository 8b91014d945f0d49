"""Round-2 ncu post-processing: the committed summaries under profiles/ from
the raw outputs of a validation script (scripts/gpu_r02fin*.sh).

usage: python scripts/ncu_summary_r02.py <tag>
  reads  gpurun_out/<tag>_launches.csv   (ncu --metrics gpu__time_duration.sum launch list)
         gpurun_out/<tag>_ga_c4_raw.csv  (ncu --set full, every ga_kernel launch of one c4 search)
         gpurun_out/<tag>_sweep_raw.csv  (ncu --set full, one sweep_kernel launch)
  writes profiles/<tag>_launches.json, profiles/<tag>_ga_c4_launches.json,
         profiles/<tag>_sweep_full.json and profiles/ncu_summary.json
         (per-launch DRAM bytes that bench.py reports as roofline.traffic)
"""
import csv
import io
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
KEYS = ["gpu__time_duration.sum", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "sass__inst_executed_local_loads", "sass__inst_executed_local_stores"]
STALL = "smsp__pcsamp_warps_issue_stalled_"
SWEEP_PLANS = 300000      # plans in the profiled sweep launch (gpu_r02fin*.sh)
BENCH_CHUNK = 1 << 21     # plans per sweep_kernel launch in bench.py


def csv_rows(path):
    text = open(path).read()
    return list(csv.reader(io.StringIO(text[text.index('"ID"'):])))


def launch_list(path):
    rows = csv_rows(path)
    h = rows[0]
    ki, mi, ui, vi = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
    agg = {}
    for r in rows[1:]:
        if r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0]
        ms = float(r[vi].replace(",", "")) * {"ms": 1.0, "us": 1e-3, "ns": 1e-6, "s": 1e3}[r[ui]]
        a = agg.setdefault(name, {"launches": 0, "ms": 0.0})
        a["launches"] += 1
        a["ms"] += ms
    tot = sum(a["ms"] for a in agg.values())
    for a in agg.values():
        a["ms"] = round(a["ms"], 3)
        a["share"] = round(a["ms"] / tot, 4)
    return dict(sorted(agg.items(), key=lambda kv: -kv[1]["ms"]))


def full_captures(path):
    rows = csv_rows(path)
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        if len(r) != len(h):
            continue
        c = {"kernel": r[h.index("Kernel Name")].split("(")[0]}
        for k in KEYS:
            if k in h:
                c[k] = f"{r[h.index(k)]} {units[h.index(k)]}".strip()
        c["dram_bytes"] = sum(float(r[h.index(k)].replace(",", "")) * SCALE[units[h.index(k)]]
                              for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        st = {k[len(STALL):]: float(r[i].replace(",", "") or 0) for i, k in enumerate(h)
              if k.startswith(STALL) and not k.endswith("not_issued")}
        c["stall_samples"] = dict(sorted(((k, v) for k, v in st.items() if v > 0), key=lambda kv: -kv[1]))
        out.append(c)
    return out


def main():
    tag = sys.argv[1]
    g = os.path.join(ROOT, "gpurun_out")
    p = os.path.join(ROOT, "profiles")
    launches = launch_list(os.path.join(g, f"{tag}_launches.csv"))
    json.dump({"command": "ncu --metrics gpu__time_duration.sum --clock-control none python bench.py "
                          "--steps 2 --warmup 1 --no-configs --no-cpu-baseline --sweep-plans 4000000 "
                          "(cold-cache, serialised: compare shares, not absolutes)",
               "kernels": launches}, open(os.path.join(p, f"{tag}_launches.json"), "w"), indent=1)
    ga = full_captures(os.path.join(g, f"{tag}_ga_c4_raw.csv"))
    json.dump({"capture": f"ncu --set full, every ga_kernel launch of one warm c4 B=10^4 search "
                          f"(scripts/gpu_{tag}.sh)", "launches": ga},
              open(os.path.join(p, f"{tag}_ga_c4_launches.json"), "w"), indent=1)
    sw = full_captures(os.path.join(g, f"{tag}_sweep_raw.csv"))[0]
    json.dump({"capture": f"ncu --set full, one sweep_kernel launch over {SWEEP_PLANS} c4 plans "
                          f"(scripts/gpu_{tag}.sh)", "launch": sw},
              open(os.path.join(p, f"{tag}_sweep_full.json"), "w"), indent=1)
    ga_bytes = [c["dram_bytes"] for c in ga]
    per_plan = sw["dram_bytes"] / SWEEP_PLANS
    summary = {"kernels": {
        "ga_kernel_c4": {"source": f"profiles/{tag}_ga_c4_launches.json: ncu --set full over every "
                                   "ga_kernel launch of one warm c4 B=10^4 search",
                         "launches": len(ga), "dram_bytes_per_launch": sum(ga_bytes) / len(ga_bytes),
                         "dram_bytes_total": sum(ga_bytes)},
        "sweep_kernel": {"source": f"profiles/{tag}_sweep_full.json: ncu --set full of one "
                                   f"sweep_kernel launch over {SWEEP_PLANS} c4 plans",
                         "plans_per_launch": SWEEP_PLANS, "dram_bytes_per_launch_profiled": sw["dram_bytes"],
                         "dram_bytes_per_plan": per_plan, "dram_bytes_per_launch": per_plan * BENCH_CHUNK,
                         "note": "scaled to the bench's 2^21-plan chunk (one sweep_kernel launch per chunk)"}}}
    json.dump(summary, open(os.path.join(p, "ncu_summary.json"), "w"), indent=1)
    print(json.dumps({"launches": launches, "ga_dram_per_launch": summary["kernels"]["ga_kernel_c4"]
                      ["dram_bytes_per_launch"], "sweep_dram_per_plan": per_plan}, indent=1))


if __name__ == "__main__":
    main()
