"""Golden per-interface sparsification ranks for the C5 generator at n=48
(3D 48^3, N=110,592, L=11, eps per CONFIGS["C5"]) from the oracle, levels
11..8 only (the oracle needs ~48 min and ~15 GB for these four levels).

Output: tests/golden/ranks_C5_n48_L8.npz, ranks[i] = (level, p, rank, before).
These levels are the first where candidate matrices exceed 65,535 columns,
the regime that exposed a grid-limit bug in the sparsify preamble.
Run from the repo root:  python tests/golden/make_n48_ranks.py
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import spaqr_oracle as O  # noqa: E402
from paper_2010_06807_b200.ordering import partition_geometric  # noqa: E402
from paper_2010_06807_b200.problems import make_config  # noqa: E402

A, dims, L, eps, b, tol = make_config("C5", n=48)
tree = partition_geometric(dims, L)
t = time.time()
F = O.factorize(A, tree, eps=eps, stop_level=8)
print("oracle levels 11..8:", round(time.time() - t, 1), "s")
r = np.array([(lev, p, rank, before) for lev, p, rank, before in F.ranks], dtype=np.int32)
np.savez_compressed(os.path.join(ROOT, "tests", "golden", "ranks_C5_n48_L8.npz"), ranks=r)
