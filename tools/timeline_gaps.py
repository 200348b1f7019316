"""Device idle gaps of the last factorization in an SPQ_SCOPE_LOG written by
tools/c3_timeline.py: sorts the scopes by start offset, reports busy time,
total idle time and the largest gaps with the scopes on either side.

    python tools/timeline_gaps.py gpurun_out/r01d/c3_scopes.txt [top]
"""
import collections
import sys

FAM = ["copy", "qr", "wy", "trsm", "cpqr", "flags", "chain"]
rows = []
for line in open(sys.argv[1]):
    if "#" in line:
        continue
    p = line.split(None, 3)
    try:
        rows.append((float(p[2]), float(p[1]), FAM[int(p[0])], p[3].strip() if len(p) > 3 else ""))
    except (ValueError, IndexError):
        pass
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
# the log holds three factorizations (scopes of one collection are contiguous)
ev = sorted(rows[2 * len(rows) // 3:])
span = ev[-1][0] + ev[-1][1]
busy = sum(e[1] for e in ev)
gaps, end, prev = [], 0.0, None
for t0, ms, f, tag in ev:
    if t0 > end:
        gaps.append((t0 - end, end, prev, (f, tag[:60])))
    end = max(end, t0 + ms)
    prev = (f, tag[:60])
print(f"span {span:.2f} ms, kernels busy {busy:.2f} ms, idle {sum(g[0] for g in gaps):.2f} ms "
      f"in {len(gaps)} gaps")
for g in sorted(gaps, reverse=True)[:top]:
    print(f"  {g[0]:7.3f} ms at {g[1]:8.2f}: {g[2]} -> {g[3]}")
h = collections.Counter()
for g in gaps:
    h[(g[2][0] if g[2] else None, g[3][0])] += g[0]
print("idle by (before, after) family:", [(k, round(v, 2)) for k, v in h.most_common(8)])
