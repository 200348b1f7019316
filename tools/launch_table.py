"""Per-kernel totals from an ncu --csv launch list (gpu__time_duration.sum)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hdr + 1:]:
    if len(r) > vi and r[mi] == "gpu__time_duration.sum":
        name = r[ki].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) / 1e3   # ns -> us
tot = sum(v[1] for v in agg.values())
for name, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{name[:70]:70s} {n:6d} {us / 1e3:9.3f} ms {us / n:9.1f} us {100 * us / tot:5.1f}%")
print("total", round(tot / 1e3, 3), "ms")
