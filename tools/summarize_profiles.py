"""Summarize a gpurun profiling batch (gpurun_out/p2) into profiles/."""
import collections
import csv
import json
import os
import subprocess
import sys

src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/p2"
dst = sys.argv[2] if len(sys.argv) > 2 else "profiles"
tag = sys.argv[3] if len(sys.argv) > 3 else "r01"
os.makedirs(dst, exist_ok=True)


def launch_summary(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.defaultdict(dict)
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        per[r[ii]]["name"] = r[ki].split("(")[0].replace("void ", "")
        try:
            per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
        except ValueError:
            pass
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for d in per.values():
        a = agg[d["name"]]
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0)
        a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    tot = sum(v[1] for v in agg.values())
    lines = ["| kernel | launches | total ms | avg us | share | DRAM bytes/launch |",
             "|---|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| {k} | {v[0]} | {v[1] / 1e6:.3f} | {v[1] / v[0] / 1e3:.1f} | "
                     f"{v[1] / tot:.1%} | {v[2] / v[0]:.3e} |")
    lines.append(f"| total | {sum(v[0] for v in agg.values())} | {tot / 1e6:.3f} | | | |")
    return "\n".join(lines)


def ncu_details(rep):
    keys = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput",
            "Achieved Occupancy", "Registers Per Thread", "Grid Size", "Block Size", "Cluster Size",
            "Dynamic Shared Memory Per Block", "Executed Ipc Active",
            "Warp Cycles Per Issued Instruction", "L2 Hit Rate"]
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    res = []
    rows_d = list(csv.reader(out.splitlines()))
    if rows_d:
        hd = rows_d[0]
        ni, ui, vi2, ki2 = hd.index("Metric Name"), hd.index("Metric Unit"), hd.index("Metric Value"), hd.index("Kernel Name")
        for r in rows_d[1:]:
            if len(r) > vi2 and r[ni] in keys:
                res.append(f"{r[ki2][:50]} | {r[ni]} | {r[vi2]} {r[ui]}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    extra = []
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    if len(rows) > 2:
        h = rows[0]
        units = rows[1]
        for v in rows[2:]:
            stalls = []
            dram = 0.0
            for i, x in enumerate(h):
                if x in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                    try:
                        dram += float(v[i].replace(",", "")) * scale.get(units[i], 1)
                    except ValueError:
                        pass
                if "smsp__pcsamp_warps_issue_stalled" in x and not x.endswith("not_issued"):
                    try:
                        stalls.append((float(v[i]), x.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                    except ValueError:
                        pass
            stalls.sort(reverse=True)
            extra.append(f"dram bytes (read+write) = {dram:.4e}; top stalls: " +
                         ", ".join(f"{n}={int(c)}" for c, n in stalls[:5]))
    return "\n".join(res + extra)


md = [f"# Profiles {tag} (B200, sm_100a)\n"]
for f in ("smi.txt",):
    p = os.path.join(src, f)
    if os.path.exists(p):
        md.append("```\n" + open(p).read().strip() + "\n```\n")
for name in ("bench.json", "bench_ref.json", "config2.json"):
    p = os.path.join(src, name)
    if os.path.exists(p):
        txt = open(p).read().strip().splitlines()
        line = txt[-1] if txt else ""
        with open(os.path.join(dst, f"{tag}_{name}"), "w") as fh:
            fh.write(line + "\n")
        md.append(f"## {name}\n```\n{line[:3000]}\n```\n")
for name in ("c4.log", "c1.log"):
    p = os.path.join(src, name)
    if os.path.exists(p):
        with open(os.path.join(dst, f"{tag}_{name}"), "w") as fh:
            fh.write(open(p).read())
lp = os.path.join(src, "launches.csv")
if os.path.exists(lp):
    md.append("## Launch list (ncu --metrics gpu__time_duration.sum,dram__bytes_*; one C3 "
              "factorization + fp64 peak probe; cold-cache, serialised: compare shares)\n")
    md.append(launch_summary(lp) + "\n")
for rep in ("prof_cpqr", "prof_gemm", "prof_panel"):
    p = os.path.join(src, rep + ".ncu-rep")
    if os.path.exists(p):
        md.append(f"## ncu --set full: {rep}\n```\n{ncu_details(p)}\n```\n")
with open(os.path.join(dst, f"{tag}_summary.md"), "w") as fh:
    fh.write("\n".join(md))
print("\n".join(md)[:6000])
