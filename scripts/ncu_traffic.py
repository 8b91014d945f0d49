"""profiles/ncu_summary.json: dram read+write bytes per launch of each kernel,
averaged over the launches of the given --set full summaries (bench.py reads
it for roofline.traffic)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def val(s):
    num, unit = s.split()
    return float(num) * SCALE[unit]


out = {"kernels": {}, "sources": []}
for spec in sys.argv[1:]:  # kernel_key=profiles/<file>_full.json
    key, path = spec.split("=")
    caps = json.load(open(os.path.join(ROOT, path)))["captures"]
    b = [val(c["dram__bytes_read.sum"]) + val(c["dram__bytes_write.sum"]) for c in caps]
    t = [float(c["gpu__time_duration.sum"].split()[0]) for c in caps]
    out["kernels"][key] = {"dram_bytes_per_launch": sum(b) / len(b), "launches": len(b),
                           "avg_launch_us": sum(t) / len(t), "source": path}
    out["sources"].append(path)
json.dump(out, open(os.path.join(ROOT, "profiles", "ncu_summary.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
