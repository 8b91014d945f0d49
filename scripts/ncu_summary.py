"""Summarise ncu outputs into profiles/ (committed evidence).

usage: python scripts/ncu_summary.py <tag> [--rep X.ncu-rep] [--launches launches.csv]
         [--kernel-name eval_kernel] [--cubin-funcs]

Writes profiles/<tag>_launches.json (per-kernel launch counts / time shares
from the gpu__time_duration launch list) and profiles/<tag>_full.json (key
metrics of the --set full capture, plus SASS stall samples aggregated per
device function when --sass-map is given).
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "gpc__cycles_elapsed.max"]


def launches(path):
    txt = open(path).read()
    start = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[start:])))
    per = {}
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
                 "msecond": 1e3}.get(unit, 1.0)
        us = v * scale
        d = per.setdefault(name, {"launches": 0, "total_us": 0.0})
        d["launches"] += 1
        d["total_us"] += us
    tot = sum(d["total_us"] for d in per.values()) or 1.0
    for d in per.values():
        d["share"] = d["total_us"] / tot
        d["avg_us"] = d["total_us"] / d["launches"]
    return {"kernels": per, "total_launches": sum(d["launches"] for d in per.values()),
            "note": "cold-cache, serialised ncu launch list: compare shares, not absolutes"}


def full(rep, sass_funcs=None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    caps = []
    for r in rows[2:]:
        d = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = r[i] + (" " + units[i] if units[i] else "")
        d["kernel"] = r[hdr.index("Kernel Name")].split("(")[0] if "Kernel Name" in hdr else ""
        caps.append(d)
    res = {"captures": caps}
    if sass_funcs:
        res["stall_samples_by_function"] = sass_by_function(rep, sass_funcs)
    return res


def sass_by_function(rep, funcs):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia, isamp = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
    iinst = hdr.index("Instructions Executed")
    base, agg = None, {}
    for r in rows[2:]:
        if len(r) <= iinst:
            continue
        try:
            a = int(r[ia], 16)
        except ValueError:
            base = None
            continue
        if base is None:
            base = a
        off = a - base
        name = "kernel_body"
        for o, n in funcs:
            if off >= o:
                name = n
        s = agg.setdefault(name, [0, 0])
        s[0] += int(float(r[isamp] or 0))
        s[1] += int(float(r[iinst] or 0))
    tot = sum(v[0] for v in agg.values()) or 1
    return {k: {"stall_samples": v[0], "share": v[0] / tot, "inst_executed": v[1]}
            for k, v in sorted(agg.items(), key=lambda x: -x[1][0])}


def cubin_funcs(obj):
    """device-function start offsets of eval_kernel's cubin (readelf symtab)."""
    tmp = "/tmp/_cubin_extract"
    os.makedirs(tmp, exist_ok=True)
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp,
                   capture_output=True)
    cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    out = subprocess.run(["readelf", "-sW", os.path.join(tmp, cub)], capture_output=True,
                         text=True).stdout
    funcs = []
    for ln in out.splitlines():
        f = ln.split()
        if len(f) >= 8 and f[3] == "FUNC" and int(f[2], 0) > 0:
            name = f[7].split("$")[-1]
            for key in ("end_to_end", "ring_small", "check_memory", "ring_heuristic",
                        "balance_data", "total_with_split", "balance_layers", "apportion",
                        "task_cost", "dblrcp", "div_rn_f64", "div_s64", "split_tables",
                        "trial", "stage_tab"):
                if key in name:
                    name = key
            funcs.append((int(f[1], 16), name))
    for f in os.listdir(tmp):
        os.remove(os.path.join(tmp, f))
    return sorted(f for f in funcs if f[0] > 0)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--rep")
    ap.add_argument("--launches")
    ap.add_argument("--obj", help="object file whose cubin maps SASS offsets to functions")
    a = ap.parse_args()
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    if a.launches:
        with open(os.path.join(ROOT, "profiles", f"{a.tag}_launches.json"), "w") as f:
            json.dump(launches(a.launches), f, indent=1)
    if a.rep:
        funcs = cubin_funcs(a.obj) if a.obj else None
        with open(os.path.join(ROOT, "profiles", f"{a.tag}_full.json"), "w") as f:
            json.dump(full(a.rep, funcs), f, indent=1)


if __name__ == "__main__":
    sys.exit(main())
