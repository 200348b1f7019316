"""Factorize + solve one config on the GPU and print timings/parity summary."""
import json
import sys
import time

sys.path.insert(0, ".")
from paper_2010_06807_b200.factor import factorize          # noqa: E402
from paper_2010_06807_b200.ordering import partition_geometric  # noqa: E402
from paper_2010_06807_b200.problems import make_config      # noqa: E402
from paper_2010_06807_b200.solve import gmres               # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
n = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2] != "-" else None
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
A, dims, L, eps, b, tol = make_config(cfg, n=n)
t0 = time.perf_counter()
tree = partition_geometric(dims, L)
print(f"tree {time.perf_counter() - t0:.2f}s N={A.ncols}", flush=True)
for r in range(reps):
    t0 = time.perf_counter()
    F = factorize(A, tree, eps=eps)
    tf = time.perf_counter() - t0
    tfac_py = tf
    tm = F.device_timings()
    t0 = time.perf_counter()
    x, rep = gmres(A, b, F, tol=tol)
    ts = time.perf_counter() - t0
    print(f"rep {r}: factor {tf:.3f}s gmres {ts:.3f}s its={rep.iterations} res={rep.final_residual:.3e}", flush=True)
    host = tm.pop("host")
    print("  device:", json.dumps({k: (round(v['ms'], 2), round(v['flops'] / 1e9, 2), v['launches']) for k, v in tm.items()}), flush=True)
    print("  host:", json.dumps({k: round(v, 2) for k, v in host.items()}), flush=True)
    print("  levels:", [(s["level"], round(s["t_factor"], 3), round(s["t_scale"], 3), round(s["t_sparsify"], 3), round(s["t_merge"], 3)) for s in F.stats], flush=True)
