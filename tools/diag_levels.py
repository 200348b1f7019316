import sys
import numpy as np
sys.path.insert(0, ".")
from paper_2010_06807_b200.factor import factorize          # noqa: E402
from paper_2010_06807_b200.ordering import partition_geometric  # noqa: E402
from paper_2010_06807_b200.problems import make_config      # noqa: E402
cfg, n = sys.argv[1], (None if sys.argv[2] == "-" else int(sys.argv[2]))
A, dims, L, eps, b, tol = make_config(cfg, n=n)
class Obs:
    def on_level(self, state, lev, st):
        print({k: (round(v, 3) if isinstance(v, float) else v) for k, v in st.items()
               if k in ("level", "n_sparsified", "fine_retired", "cols_after", "trailing_blocks",
                        "t_factor", "t_sparsify", "_live_gb", "_peak_gb")}, flush=True)


F = factorize(A, partition_geometric(dims, L), eps=eps, _memstats=True, observer=Obs())
for s in F.stats:
    print({k: (round(v, 3) if isinstance(v, float) else v) for k, v in s.items()
           if k in ("level", "cols_before", "n_factored", "factored_cols", "n_scaled", "n_sparsified",
                    "fine_retired", "iface_max", "cols_after", "trailing_blocks", "t_factor", "t_sparsify", "_live_gb", "_peak_gb")})
log = np.array(F.sparsify_log)
for lev in sorted(set(log[:, 0]), reverse=True):
    sel = log[log[:, 0] == lev]
    print("lev", lev, "n", len(sel), "before(min/med/max)", sel[:, 2].min(), int(np.median(sel[:, 2])), sel[:, 2].max(),
          "rank(min/med/max)", sel[:, 3].min(), int(np.median(sel[:, 3])), sel[:, 3].max())
