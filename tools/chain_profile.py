"""Per-wave device times of solve_w / apply_w (SPQ_CHAIN_PROFILE=1). Diagnostic."""
import os
import sys

os.environ["SPQ_CHAIN_PROFILE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2010_06807_b200.factor import factorize  # noqa: E402
from paper_2010_06807_b200.ordering import partition_geometric  # noqa: E402
from paper_2010_06807_b200.problems import make_config  # noqa: E402

A, dims, L, eps, b, tol = make_config(sys.argv[1] if len(sys.argv) > 1 else "C3")
F = factorize(A, partition_geometric(dims, L), eps=eps)
y = np.random.default_rng(0).standard_normal(A.ncols)
for _ in range(2):
    F.apply_qt(y)
    F.solve_w(y)
    F.apply_w(y)
