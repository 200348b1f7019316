"""Run one config through the device path and print timings.

    python tools/run_config.py CFG [n|-] [reps] [levels]

Diagnostic driver (not part of the product): factorize + device GMRES,
per-level wall times from the observer hook."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2010_06807_b200.factor import factorize  # noqa: E402
from paper_2010_06807_b200.ordering import partition_geometric  # noqa: E402
from paper_2010_06807_b200.problems import make_config  # noqa: E402
from paper_2010_06807_b200.solve import gmres  # noqa: E402

cfg = sys.argv[1]
n = None if len(sys.argv) < 3 or sys.argv[2] == "-" else int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
levels = int(sys.argv[4]) if len(sys.argv) > 4 else None
A, dims, L, eps, b, tol = make_config(cfg, n=n, levels=levels)
tree = partition_geometric(dims, L)
print(f"{cfg} n={n} N={A.ncols} L={L} eps={eps}", flush=True)
t_last = [time.perf_counter()]


class Obs:
    F = None
    prev = {}

    def on_level(self, state, lev, st):
        t = time.perf_counter()
        dev = ""
        if Obs.ctx is not None:
            tm = Obs.ctx.timings()
            cur = {k: v["ms"] for k, v in tm.items() if k != "host"}
            d = {k: cur[k] - Obs.prev.get(k, 0.0) for k in cur}
            Obs.prev = cur
            dev = " dev[" + " ".join(f"{k}={v:.1f}" for k, v in d.items() if v > 0.05) + \
                f"] sum={sum(d.values()):.1f}ms"
        keys = ("n_factored", "n_scaled", "n_sparsified", "fine_retired", "cols_after",
                "trailing_blocks", "t_factor", "t_scale", "t_sparsify")
        print(f"  level {lev}: {t - t_last[0]:.3f} s "
              + " ".join(f"{k}={st[k]:.3f}" if isinstance(st.get(k), float) else f"{k}={st.get(k)}"
                         for k in keys if k in st) + dev, flush=True)
        t_last[0] = t


obs = Obs()
Obs.ctx = None
_Ctx = None
import paper_2010_06807_b200.factor as _FZ  # noqa: E402
_orig_ctx = _FZ.Context


class _SpyCtx(_orig_ctx):
    def __init__(self, *a, **k):
        super().__init__(*a, **k)
        Obs.ctx = self
        Obs.prev = {}


_FZ.Context = _SpyCtx


for r in range(reps):
    t0 = time.perf_counter()
    t_last[0] = t0
    F = factorize(A, tree, eps=eps, observer=obs if r == reps - 1 else None)
    t1 = time.perf_counter()
    print(f"factor {t1 - t0:.3f} s", flush=True)
x, rep = gmres(A, b, F, tol=tol)
t2 = time.perf_counter()
x, rep = gmres(A, b, F, tol=tol)
t3 = time.perf_counter()
print(f"gmres {t3 - t2:.3f} s its={rep.iterations} res={rep.final_residual:.3e} "
      f"conv={rep.converged}", flush=True)
print("ranks", [r for _, _, _, r in F.sparsify_log][:40])
if os.environ.get("SPQ_TIMINGS"):
    # last factorization (no observer): device families + host breakdown
    F = factorize(A, tree, eps=eps, _marks=True)
    tm = F.device_timings()
    print(f"device_ms(marks)={F.device_ms:.2f}")
    for k, v in tm.items():
        if k == "host":
            print("host", {a: (round(b, 2) if isinstance(b, float) else b) for a, b in v.items()})
        elif v["ms"]:
            print(f"  {k:8s} {v['ms']:9.2f} ms {v['flops'] / 1e9:9.3f} GF {v['launches']:6d} launches")
