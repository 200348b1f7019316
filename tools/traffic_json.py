"""ncu launch list (gpu__time_duration.sum + dram__bytes_{read,write}.sum, --csv) ->
profiles/ncu_traffic.json: per kernel and per bench kernel family, launches, average
duration and DRAM bytes (read+write) per launch.  bench.py reads the family figure
into roofline.traffic.

usage: python tools/traffic_json.py gpurun_out/r01c/launches.csv profiles/ncu_traffic.json
"""
import collections
import csv
import json
import sys

# bench.py kernel families (runtime.cu Fam scopes) -> kernel-name prefixes
FAMILIES = {
    "cpqr": ("cpqr_", "sparsify_select_kernel", "colsq_kernel", "gather_cols_kernel",
             "select_batch_kernel", "colsq_batch_kernel", "gather_cols_batch_kernel"),
    "qr": ("panel_qr", "larft", "pivot_check_kernel"),
    "wy": ("gemm_dmma", "wyf_kernel", "splitk_reduce_kernel"),
    "trsm": ("trsm_",),
    "copy": ("copy_tasks_kernel",),
    "flags": ("rowflags", "count_nnz_kernel"),
    "chain": ("chain_",),
}


def family(name):
    for f, prefixes in FAMILIES.items():
        if name.startswith(prefixes):
            return f
    return None


def main(src, dst):
    rows = list(csv.reader(open(src)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi, ii = (h.index("Kernel Name"), h.index("Metric Name"),
                      h.index("Metric Value"), h.index("ID"))
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        names[r[ii]] = r[ki].split("(")[0].replace("void ", "").split("<")[0].replace("spq::", "")
        per[r[ii]][r[mi]] = float(r[vi].replace(",", ""))
    kern = collections.defaultdict(lambda: {"launches": 0, "us": 0.0, "dram_bytes": 0.0})
    for lid, m in per.items():
        k = kern[names[lid]]
        k["launches"] += 1
        k["us"] += m.get("gpu__time_duration.sum", 0.0) / 1e3
        k["dram_bytes"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    fam = collections.defaultdict(lambda: {"launches": 0, "us": 0.0, "dram_bytes": 0.0})
    for n, k in kern.items():
        f = family(n)
        if f:
            for key in k:
                fam[f][key] += k[key]
    out = {"source": src,
           "note": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                   "--clock-control none (cold-cache, serialised launches)",
           "kernels": {n: {"launches": k["launches"], "avg_us": k["us"] / k["launches"],
                           "dram_bytes_per_launch": k["dram_bytes"] / k["launches"]}
                       for n, k in sorted(kern.items(), key=lambda kv: -kv[1]["us"])},
           "families": {f: {"launches": v["launches"], "avg_us": v["us"] / v["launches"],
                            "dram_bytes_per_launch": v["dram_bytes"] / v["launches"]}
                        for f, v in fam.items() if v["launches"]}}
    json.dump(out, open(dst, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
