"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel."""
import csv, sys
from collections import defaultdict
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
ui = h.index("Metric Unit")
agg = defaultdict(list)
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    v = {"ns": v / 1e6, "us": v / 1e3, "usecond": v / 1e3, "ms": v, "msecond": v, "nsecond": v / 1e6}.get(r[ui], v)
    name = r[ki].split("(")[0]
    agg[name].append(v)
tot = sum(sum(v) for v in agg.values())
print("| kernel | launches | mean ms | total ms | share of our kernel time |")
print("|---|---|---|---|---|")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"| {k} | {len(v)} | {sum(v)/len(v):.4f} | {sum(v):.3f} | {100*sum(v)/tot:.1f}% |")
