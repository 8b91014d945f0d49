"""Per-plan sub-phase averages from HPG_PLAN_PROFILE output (diagnostics)."""
import gzip
import sys

NAMES = {0: "bl.geometry", 1: "bl.others_fit", 2: "bl.exact_fill", 3: "bl.exact_trials",
         4: "bl.exact_set", 5: "bl.greedy_init", 6: "bl.greedy_bottleneck", 7: "bl.greedy_fill",
         8: "bl.greedy_trials", 9: "bl.greedy_set", 10: "bl.check_memory", 12: "geometry",
         13: "geometry.tp_rings", 14: "geometry.pp_pairs", 15: "task_cost.dp_rings",
         16: "task_cost", 17: "end_to_end", 20: "class_costs", 21: "ring_bottleneck",
         22: "e2e.resident", 23: "e2e.bridge"}
rows = [l.split() for l in gzip.open(sys.argv[1], "rt")]
for lab, cond in (("waves<=32", lambda n: n <= 32), ("all", lambda n: True)):
    acc = [0] * 4
    sub = [0] * 27
    cnt = 0
    for r in rows:
        if not cond(int(r[1])):
            continue
        p = [int(x) for x in r[4:8]]
        bar = r.index("|")
        s = [int(x) for x in r[bar + 1:]]
        cnt += 1
        for i in range(4):
            acc[i] += p[i]
        for i in range(min(27, len(s))):
            sub[i] += s[i]
    print(lab, cnt, "plans; avg cycles stage/balance_data/balance_layers/final",
          [a // cnt for a in acc])
    for i in range(27):
        if sub[i]:
            print(f"   {i:2d} {NAMES.get(i, '?'):24s} {sub[i] // cnt}")
