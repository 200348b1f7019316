"""Per-kernel summary of an ncu counter CSV (tools/gpu_counters.sh):
launches, total/avg time, achieved DRAM GB/s, DMMA and FP64 pipe % (time-weighted)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
L = collections.defaultdict(dict)
for r in rows[hdr + 1:]:
    if len(r) > vi:
        L[int(r[ii])][r[mi]] = float(r[vi].replace(",", "")) if r[vi].replace(",", "").replace(".", "").isdigit() else r[vi]
        L[int(r[ii])]["name"] = r[ki].split("(")[0].replace("void ", "").replace("spq::", "")
agg = collections.defaultdict(lambda: collections.Counter())
for d in L.values():
    t = d.get("gpu__time_duration.sum", 0.0)
    if not isinstance(t, float):
        continue
    a = agg[d["name"][:44]]
    a["n"] += 1
    a["ns"] += t
    a["bytes"] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    a["dmma"] += t * d.get("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed", 0.0)
    a["fp64"] += t * d.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed", 0.0)
tot = sum(a["ns"] for a in agg.values())
print(f"| kernel | launches | total ms | avg us | share | DRAM GB/s | DMMA pipe % | FP64 pipe % |")
print("|---|---|---|---|---|---|---|---|")
for name, a in sorted(agg.items(), key=lambda kv: -kv[1]["ns"])[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"| {name} | {a['n']} | {a['ns'] / 1e6:.3f} | {a['ns'] / a['n'] / 1e3:.1f} | {100 * a['ns'] / tot:.1f}% | "
          f"{a['bytes'] / a['ns']:.1f} | {a['dmma'] / a['ns']:.1f} | {a['fp64'] / a['ns']:.1f} |")
print(f"| total | {sum(a['n'] for a in agg.values())} | {tot / 1e6:.3f} | | | | | |")
