"""Instruction count of eval_kernel's SASS per source function (diagnostics)."""
import collections
import re
import subprocess
import sys

cubin = sys.argv[1]
sass = subprocess.run(["nvdisasm", "--print-line-info", cubin], capture_output=True,
                      text=True).stdout
cur = None
cnt = collections.Counter()
for l in sass.splitlines():
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    if re.search(r"/\*[0-9a-f]{4,}\*/", l) and cur:
        cnt[cur] += 1
base = "/root/repo/paper_2512_12476_b200/csrc/"


def funcs(path):
    out = []
    for i, l in enumerate(open(path).read().split("\n"), 1):
        m = re.match(r"(?:__device__|__global__|HPG_HD|template).*?(\w+)\(", l)
        if m and not l.strip().endswith(";"):
            out.append((i, m.group(1)))
    return out


F = {f: funcs(base + f) for f in ("eval.cu", "eval_device.cuh", "common.hpp", "rng.hpp")}
agg = collections.Counter()
for (f, line), n in cnt.items():
    name = "?"
    for (i, nm) in F.get(f, []):
        if i <= line:
            name = nm
    agg[(f, name)] += n
print("total", sum(agg.values()))
for k, v in agg.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30):
    print(v, k)
