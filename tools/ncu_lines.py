"""Top CUDA source lines of an ncu report by warp-stall samples, with the
dominant stall reasons per line.   python tools/ncu_lines.py REP [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
h = rows[hdr]
si = h.index("Warp Stall Sampling (All Samples)")
stall_cols = [(i, n) for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
lines = []
cur = None
for r in rows[hdr + 1:]:
    if len(r) <= si:
        continue
    if r[0]:   # a CUDA source line (aggregate of its SASS)
        try:
            s = int(r[si])
        except ValueError:
            continue
        st = sorted(((int(r[i]) if i < len(r) and r[i].isdigit() else 0, n[6:]) for i, n in stall_cols), reverse=True)[:3]
        lines.append((s, r[0], r[1].strip()[:80], st))
tot = sum(l[0] for l in lines)
print(f"total samples {tot}")
for s, ln, src, st in sorted(lines, reverse=True)[:top]:
    print(f"{s:6d} {100 * s / max(tot, 1):5.1f}% L{ln:5s} {src:80s} " + " ".join(f"{n}={v}" for v, n in st if v))
