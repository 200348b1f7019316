"""Size sweep of the factorization (is O(N log N) preserved?).

    python tools/scaling_sweep.py OUT.json [--oracle-budget SECONDS]

2D: the C3 generator (variable kappa, random beta, eps 1e-3) at n = 64..512;
3D: the C5 generator (variable kappa, random beta, eps 1e-2) at n = 16..64 and
the C4 generator (constant coefficients, eps 1e-2) at n = 16..40; L =
ceil(log2(N/64)) except the BASELINE points (C3 L=10, C4 L=9, C5 L=11).
Per point: device time of a warm factorization (median of 3, load-inclusive
marks, clocks sampled), per-level host phase times, interface-size
statistics, payload, and the CPU oracle's time where it fits the budget.
Fitted exponents (log time vs log N) per family are appended."""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2010_06807_b200.factor import factorize  # noqa: E402
from paper_2010_06807_b200.ordering import partition_geometric  # noqa: E402
from paper_2010_06807_b200.problems import default_levels, make_config  # noqa: E402

out_path = sys.argv[1]
budget = 60.0
if "--oracle-budget" in sys.argv:
    budget = float(sys.argv[sys.argv.index("--oracle-budget") + 1])
fams = {
    "2d_var (C3 gen)": ("C3", [64, 96, 128, 192, 256, 384, 512], {256: 10}),
    "3d_var (C5 gen)": ("C5", [16, 24, 32, 40, 48, 64], {64: 11}),
    "3d_const (C4 gen)": ("C4", [16, 24, 32, 40], {32: 9}),
}
res = {"points": [], "fits": {}}
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
for fam, (cfg, ns, fixed) in fams.items():
    for n in ns:
        A, dims, L, eps, b, tol = make_config(cfg, n=n, levels=fixed.get(n))
        tree = partition_geometric(dims, L)
        times, walls = [], []
        F = None
        import gc
        gc.collect()
        try:
            for r in range(4 if A.ncols <= 100000 else 2):
                F = None
                gc.collect()
                t0 = time.perf_counter()
                F = factorize(A, tree, eps=eps, _marks=True)
                walls.append(time.perf_counter() - t0)
                times.append(F.device_ms)
        except Exception as e:   # a point that does not fit is reported, not fatal
            pt = {"family": fam, "config": cfg, "n": n, "N": int(A.ncols), "L": int(L),
                  "failed": str(e)[:300]}
            res["points"].append(pt)
            print(json.dumps(pt), flush=True)
            json.dump(res, open(out_path, "w"), indent=1)
            continue
        dev = float(np.median(times[1:]))
        tm = F.device_timings()
        host = tm.pop("host")
        pt = {"family": fam, "config": cfg, "n": n, "N": int(A.ncols), "L": int(L), "eps": eps,
              "device_ms": dev, "wall_ms": 1e3 * float(np.median(walls[1:])),
              "spec_retries": int(getattr(F, "spec_retries", 0)),
              "gflop": sum(v.get("flops", 0.0) for v in tm.values()) / 1e9,
              "family_ms": {k: round(v.get("ms", 0.0), 2) for k, v in tm.items()},
              "sparsify_waves": int(host.get("sparsify_waves", 0)),
              "syncs": int(host.get("syncs", 0)), "kernels": int(host.get("kernels", 0)),
              "peak_gb": host.get("peak_bytes", 0) / 1e9,
              "payload_scalars": int(F.payload_scalars),
              "iface_max": max(int(s["iface_max"]) for s in F.stats),
              "cols_after_last_sparsified": [int(s["cols_after"]) for s in F.stats],
              "t_phase_ms": {k: 1e3 * sum(s[k] for s in F.stats)
                             for k in ("t_factor", "t_scale", "t_sparsify", "t_merge")}}
        del F
        if budget > 0:
            try:
                from oracle import spaqr_oracle as O
                est = res.get("_last_oracle", {}).get(fam)
                if est is None or est * 4 < budget:
                    t0 = time.perf_counter()
                    O.factorize(A, tree, eps=eps)
                    ot = time.perf_counter() - t0
                    pt["oracle_s"] = ot
                    res.setdefault("_last_oracle", {})[fam] = ot
            except MemoryError:
                pt["oracle_s"] = None
        res["points"].append(pt)
        print(json.dumps(pt), flush=True)
        json.dump(res, open(out_path, "w"), indent=1)
for fam in fams:
    pts = [p for p in res["points"] if p["family"] == fam and "device_ms" in p]
    if len(pts) >= 3:
        x = np.log([p["N"] for p in pts])
        y = np.log([p["device_ms"] for p in pts])
        slope = float(np.polyfit(x, y, 1)[0])
        xs = np.log([p["N"] * math.log(p["N"]) for p in pts])
        res["fits"][fam] = {"payload_exponent_N": float(np.polyfit(
                                x, np.log([p["payload_scalars"] for p in pts]), 1)[0]),
                            "gflop_exponent_N": float(np.polyfit(
                                x, np.log([max(p["gflop"], 1e-9) for p in pts]), 1)[0]),
                            "exponent_N": slope,
                            "exponent_NlogN": float(np.polyfit(xs, y, 1)[0]),
                            "last3_exponent_N": float(np.polyfit(x[-3:], y[-3:], 1)[0])}
        po = [p for p in pts if p.get("oracle_s")]
        if len(po) >= 3:
            res["fits"][fam]["oracle_exponent_N"] = float(np.polyfit(
                np.log([p["N"] for p in po]), np.log([p["oracle_s"] for p in po]), 1)[0])
res.pop("_last_oracle", None)
json.dump(res, open(out_path, "w"), indent=1)
print(json.dumps(res["fits"], indent=1))
