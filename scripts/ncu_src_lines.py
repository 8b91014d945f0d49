"""Stall samples per CUDA source line from `ncu --page source --csv
--print-source cuda,sass` output (diagnostics)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
cur_file, agg, tot = None, {}, 0
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0] != "" and r[0] != "-":
        line, src = r[0], r[1]
        try:
            s = int(r[4])
        except ValueError:
            s = 0
        key = (cur_file, int(line))
        agg[key] = (agg.get(key, (0, src))[0] + s, src)
        tot += s
print("total samples", tot)
byfile = {}
for (f, l), (s, src) in agg.items():
    byfile[f] = byfile.get(f, 0) + s
for f, s in sorted(byfile.items(), key=lambda x: -x[1]):
    print(f"{s:8d} {100*s/max(1,tot):5.1f}%  {f}")
for (f, l), (s, src) in sorted(agg.items(), key=lambda x: -x[1][0])[:top]:
    print(f"{s:7d} {100*s/max(1,tot):5.1f}% {f}:{l}  {src.strip()[:90]}")
