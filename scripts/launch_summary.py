"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = collections.OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) <= vi or not r[vi]: continue
    v = float(r[vi].replace(",", ""))
    unit = r[ui]
    ms = v / 1e6 if unit == "ns" else v / 1e3 if unit in ("us", "usecond") else v if unit in ("ms", "msecond") else v / 1e6
    name = r[ki].split("(")[0][:70]
    a = agg.setdefault(name, [0, 0.0]); a[0] += 1; a[1] += ms
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':72s} {'launches':>8s} {'ms total':>10s} {'share':>6s}")
for k, (n, ms) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:72s} {n:8d} {ms:10.3f} {100*ms/tot:5.1f}%")
print(f"{'TOTAL':72s} {sum(a[0] for a in agg.values()):8d} {tot:10.3f}")
