"""Size-independent checks of a factorization: chain consistency and (with
eps=0, no sparsification) exactness of P^T Q^T A W^-1 = I on random vectors."""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2010_06807_b200.factor import factorize          # noqa: E402
from paper_2010_06807_b200.ordering import partition_geometric  # noqa: E402
from paper_2010_06807_b200.problems import make_config      # noqa: E402
from paper_2010_06807_b200.sparse import matvec             # noqa: E402

cfg, n = sys.argv[1], int(sys.argv[2])
exact = len(sys.argv) > 3 and sys.argv[3] == "exact"
A, dims, L, eps, b, tol = make_config(cfg, n=n)
tree = partition_geometric(dims, L)
F = factorize(A, tree, eps=0.0 if exact else eps, sparsify=not exact)
rng = np.random.default_rng(0)
y = rng.standard_normal(A.ncols)
e1 = np.linalg.norm(F.apply_w(F.solve_w(y)) - y) / np.linalg.norm(y)
e2 = abs(np.linalg.norm(F.apply_qt(y)) - np.linalg.norm(y)) / np.linalg.norm(y)
e3 = np.linalg.norm(F.apply_qt(matvec(A, F.solve_w(y))) - y) / np.linalg.norm(y)
print(f"{cfg} n={n} exact={exact} W-roundtrip={e1:.2e} Qt-isometry={e2:.2e} PtQtAWinv-I={e3:.2e}", flush=True)
