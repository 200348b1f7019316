"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck /
synccheck): factorization (scaled and unscaled routes), chains, device
GMRES, and the batched config-2 kernels, at sizes that finish under the
tools' slowdown.  Diagnostic driver."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2010_06807_b200.factor import factorize  # noqa: E402
from paper_2010_06807_b200.ordering import partition_geometric  # noqa: E402
from paper_2010_06807_b200.problems import make_config  # noqa: E402
from paper_2010_06807_b200.solve import gmres  # noqa: E402

cases = [("C1", 24, {}), ("C3", 48, {}), ("C4", 12, {}), ("C3", 48, {"mode": "unscaled"})]
if len(sys.argv) > 1 and sys.argv[1] == "quick":
    cases = cases[:2]
for cfg, n, opts in cases:
    A, dims, L, eps, b, tol = make_config(cfg, n=n)
    F = factorize(A, partition_geometric(dims, L), eps=eps, **opts)
    x, rep = gmres(A, b, F, tol=tol)
    y = np.random.default_rng(0).standard_normal((A.ncols, 2))
    F.apply_w(F.solve_w(y))
    print(cfg, n, opts, "its", rep.iterations, "res", f"{rep.final_residual:.2e}", flush=True)
from paper_2010_06807_b200.batched import batched_qr, batched_rrqr, config2_inputs  # noqa: E402
Bs, Cs, Ms = config2_inputs(n_qr=24, n_rrqr=8)
batched_qr(Bs, Cs)
batched_rrqr(Ms, 1e-2)
print("ok", flush=True)
