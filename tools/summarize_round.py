"""Write a profiles/<tag>_summary.md from a gpurun_out/<dir> produced by
tools/gpu_round.sh (bench line, reference arm, launch table, ncu highlights).

    python tools/summarize_round.py gpurun_out/r1b profiles/r01b
"""
import collections
import csv
import json
import os
import subprocess
import sys

src, dst = sys.argv[1], sys.argv[2]
out = [f"# Profiles {os.path.basename(dst)} (B200, sm_100a)\n"]
if os.path.exists(f"{src}/gpu.txt"):
    out += ["```", open(f"{src}/gpu.txt").read().strip(), "```\n"]
for name in ("bench.json", "bench_ref.json"):
    p = f"{src}/{name}"
    if os.path.exists(p):
        txt = open(p).read().strip().splitlines()
        if txt:
            out += [f"## {name}", "```", txt[-1], "```\n"]
            open(f"{dst}_{name}", "w").write(txt[-1] + "\n")
p = f"{src}/launches.csv"
if os.path.exists(p):
    rows = list(csv.reader(open(p)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    L = collections.defaultdict(dict)
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            try:
                L[int(r[ii])][r[mi]] = float(r[vi].replace(",", ""))
            except ValueError:
                pass
            L[int(r[ii])]["name"] = r[ki].split("(")[0].replace("void ", "").replace("spq::", "")[:60]
    agg = collections.defaultdict(collections.Counter)
    for d in L.values():
        t = d.get("gpu__time_duration.sum", 0.0)
        a = agg[d["name"]]
        a["n"] += 1
        a["ns"] += t
        a["b"] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    tot = sum(a["ns"] for a in agg.values())
    out += ["## Launch list (ncu --metrics gpu__time_duration.sum,dram__bytes_{read,write}.sum "
            "--clock-control none; `bench.py --steps 1 --warmup 0`: fp64 peak probe + one C3 "
            "factorization + the solve-phase factorization, first 4000 launches; cold-cache and "
            "serialised: compare shares)\n",
            "| kernel | launches | total ms | avg us | share | DRAM GB/s |", "|---|---|---|---|---|---|"]
    for n, a in sorted(agg.items(), key=lambda kv: -kv[1]["ns"])[:24]:
        out.append(f"| {n} | {a['n']} | {a['ns'] / 1e6:.2f} | {a['ns'] / a['n'] / 1e3:.1f} | "
                   f"{100 * a['ns'] / tot:.1f}% | {a['b'] / max(a['ns'], 1):.1f} |")
    out.append(f"| total | {sum(a['n'] for a in agg.values())} | {tot / 1e6:.2f} | | | |\n")
KEYS = ("Duration", "Registers Per Thread", "Block Size", "Grid Size", "Cluster Size",
        "Achieved Occupancy", "Executed Ipc Active", "DRAM Throughput", "Memory Throughput",
        "Compute (SM) Throughput", "Dynamic Shared Memory Per Block")
for rep in sorted(f for f in os.listdir(src) if f.endswith(".ncu-rep")):
    path = f"{src}/{rep}"
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(det.splitlines()))
    lines = []
    kname = ""
    if rows:
        hh = rows[0]
        ni, ui, vv = hh.index("Metric Name"), hh.index("Metric Unit"), hh.index("Metric Value")
        seen = set()
        for r in rows[1:]:
            if len(r) > vv and r[ni] in KEYS and r[ni] not in seen:
                seen.add(r[ni])
                kname = r[4]
                lines.append(f"{r[ni]} = {r[vv]} {r[ui]}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics",
                          "dram__bytes_read.sum,dram__bytes_write.sum"], capture_output=True,
                         text=True).stdout
    out += [f"## ncu --set full: {rep}", f"kernel: {kname.split('(')[0]}", "```"] + lines + ["```"]
    rr = list(csv.reader(raw.splitlines()))
    if len(rr) >= 3:
        try:
            hh = rr[0]
            b = sum(float(rr[2][hh.index(m)].replace(",", "")) for m in
                    ("dram__bytes_read.sum", "dram__bytes_write.sum") if m in hh)
            out.append(f"dram bytes (read+write) per launch: {b:.4g}\n")
        except (ValueError, IndexError):
            pass
    top = subprocess.run([sys.executable, "tools/ncu_lines.py", path, "8"], capture_output=True,
                         text=True).stdout
    out += ["top stall lines:", "```", top.strip(), "```\n"]
open(f"{dst}_summary.md", "w").write("\n".join(out) + "\n")
print("wrote", f"{dst}_summary.md")
