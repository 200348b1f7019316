"""Per-level host wall times (t_factor / t_scale / t_sparsify / t_merge of the
stats) of a warm factorization, plus the device-timed total.  Diagnostic."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_06807_b200.factor import factorize  # noqa: E402
from paper_2010_06807_b200.ordering import partition_geometric  # noqa: E402
from paper_2010_06807_b200.problems import make_config  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C3"
A, dims, L, eps, b, tol = make_config(cfg)
tree = partition_geometric(dims, L)
for r in range(4):
    F = factorize(A, tree, eps=eps, _marks=True)
print(f"{cfg}: device {F.device_ms:.2f} ms")
tot = {}
for st in F.stats:
    row = {k: 1e3 * st[k] for k in ("t_factor", "t_scale", "t_sparsify", "t_merge")}
    for k, v in row.items():
        tot[k] = tot.get(k, 0.0) + v
    print(f"level {st['level']:2d}: " + "  ".join(f"{k[2:]} {v:7.2f}" for k, v in row.items())
          + f"  factored {st['n_factored']} sparsified {st['n_sparsified']}")
print("total: " + "  ".join(f"{k[2:]} {v:7.2f}" for k, v in tot.items()))
h = F.device_timings()["host"]
print({k: round(v, 2) if isinstance(v, float) else v for k, v in h.items()})
