"""Summarise HPG_PLAN_PROFILE output (diagnostics)."""
import collections
import gzip
import sys

rows = [l.split() for l in gzip.open(sys.argv[1], "rt")]
ph = [0, 0, 0, 0]
recs = []
for r in rows:
    w, n, ms, mode = int(r[0]), int(r[1]), float(r[2]), int(r[3])
    p = [int(x) for x in r[4:8]]
    for i in range(4):
        ph[i] += p[i]
    bar = r.index("|") if "|" in r else len(r)
    sub = [int(x) for x in r[bar + 1:]]
    recs.append((sum(p), mode, p, r[8:bar], w, n, ms, sub))
print(len(rows), "plans; phase totals (Gcyc) stage,bd,bl,e2e", [round(x / 1e9, 3) for x in ph])
recs.sort(reverse=True)
for x in recs[:int(sys.argv[2]) if len(sys.argv) > 2 else 12]:
    print(" ", x)
wav = collections.defaultdict(list)
for x in recs:
    wav[x[4]].append(x)
print("waves by ms:")
for w, l in sorted(wav.items(), key=lambda kv: -kv[1][0][6])[:8]:
    print("  wave", w, "n", len(l), "ms", l[0][6], "max cyc", max(x[0] for x in l),
          "sum Gcyc", round(sum(x[0] for x in l) / 1e9, 3))
tot_ms = sum(l[0][6] for l in wav.values())
print("total ms", round(tot_ms, 2), "waves", len(wav))
