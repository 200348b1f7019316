"""Per-phase clock64 breakdown of a pivot step of the register CPQR kernel
(library built with SPQ_TRACE=1): stamps of the LAST CPQR launch of a
factorization (the top sparsified level). Diagnostic only.

    SPQ_TRACE=1 python -m paper_2010_06807_b200.build --force && python tools/cpqr_trace.py
"""
import ctypes as C
import os
import sys

import numpy as np

os.environ.pop("SPQ_CPQR_LOG", None)
sys.path.insert(0, ".")
from paper_2010_06807_b200._lib import load_library  # noqa: E402
from paper_2010_06807_b200.factor import factorize  # noqa: E402
from paper_2010_06807_b200.ordering import partition_geometric  # noqa: E402
from paper_2010_06807_b200.problems import make_config  # noqa: E402

lib = load_library()
names = ["wait", "winner", "sigma", "scalars+v", "barrier F", "dots", "update+norms", "stage", "push"]
for cfg, n in (("C3", None), ("C3", 128), ("C4", 16)):
    A, dims, L, eps, b, tol = make_config(cfg, n=n)
    tree = partition_geometric(dims, L)
    for rep in range(2):
        F = factorize(A, tree, eps=eps)
    buf = np.zeros(64 * 12, np.int64)
    lib.spq_debug_cpqr_trace(buf.ctypes.data_as(C.POINTER(C.c_longlong)), buf.size)
    t = buf.reshape(64, 12)
    rank = F.sparsify_log[-1][3]
    steps = max(4, min(rank - 2, 60))
    d = np.diff(t[2:steps, :10], axis=1)
    per = np.diff(t[2:steps, 0])
    print(f"{cfg} n={n}: last interface {F.sparsify_log[-1]}: cycles/step {per.mean():.0f} "
          f"({per.mean() / 1.965e3:.2f} us)", flush=True)
    for k, nm in enumerate(names):
        print(f"   {nm:22s} {d[:, k].mean():8.0f}")
    print(f"   {'loop back':14s} {(t[3:steps, 0] - t[2:steps - 1, 9]).mean():8.0f}", flush=True)
    del F
