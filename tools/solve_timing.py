"""Solve-phase timing: device-timed chain applications and the host GMRES."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2010_06807_b200.factor import factorize          # noqa: E402
from paper_2010_06807_b200.ordering import partition_geometric  # noqa: E402
from paper_2010_06807_b200.problems import make_config      # noqa: E402
from paper_2010_06807_b200.solve import gmres               # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
A, dims, L, eps, b, tol = make_config(cfg)
F = factorize(A, partition_geometric(dims, L), eps=eps)
y = np.random.default_rng(0).standard_normal(A.ncols)
out = {}
for w, name in enumerate(("apply_qt", "solve_w", "apply_w")):
    info = np.zeros(4, np.int64)
    F._ctx.call("spq_chain_info", w, info)
    out[name + "_program"] = {"waves": int(info[0]), "ops": int(info[1]), "max_ops_per_wave": int(info[2]), "kmax": int(info[3])}
for fn in ("apply_qt", "solve_w", "apply_w"):
    getattr(F, fn)(y)                    # first call compiles the wave program + graph
    F._ctx.call("spq_reset_timings")
    t0 = time.perf_counter()
    for _ in range(10):
        getattr(F, fn)(y)
    out[fn + "_host_ms"] = (time.perf_counter() - t0) / 10 * 1e3
    out[fn + "_device_ms"] = F.device_timings()["chain"]["ms"] / 10
t0 = time.perf_counter()
x, rep = gmres(A, b, F, tol=tol)
out["gmres_s"] = time.perf_counter() - t0
out["gmres_its"] = rep.iterations
out["gmres_apply_s"] = rep.t_apply
out["final_res"] = rep.final_residual
print(json.dumps(out))
