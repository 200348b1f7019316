"""Golden symbolic fill patterns from the LIVE reference
(`nestqr.factor.symbolic_fill_levels`, factor.py:1004-1050) for C1@24^2,
C3@48^2 and C4@12^3: per level the sorted (row cid, col cid) pairs.
Run in the build container:  python tests/golden/make_symbolic.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
from nestqr.factor import symbolic_fill_levels as ref_symbolic  # noqa: E402
from nestqr.sparse import SparseMat  # noqa: E402

from paper_2010_06807_b200.ordering import partition_geometric  # noqa: E402
from paper_2010_06807_b200.problems import make_config  # noqa: E402

out = {}
for cfg, n in (("C1", 24), ("C3", 48), ("C4", 12)):
    A, dims, L, eps, b, tol = make_config(cfg, n=n)
    tree = partition_geometric(dims, L)
    Ar = SparseMat(A.nrows, A.ncols, A.indptr, A.indices, A.data)
    pat = ref_symbolic(Ar, tree)
    for lev, pairs in pat.items():
        out[f"{cfg}_n{n}_L{lev}"] = np.array(sorted(pairs), np.int32).reshape(-1, 2)
np.savez_compressed(os.path.join(ROOT, "tests", "golden", "symbolic.npz"), **out)
print({k: v.shape for k, v in out.items()})
