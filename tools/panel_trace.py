"""Per-phase clock64 breakdown of a column step of the register panel QR
kernel (library built with SPQ_TRACE=1); stamps of the last panel launch of
`qr_house` on a few shapes. Diagnostic only."""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2010_06807_b200 import kernels as K  # noqa: E402
from paper_2010_06807_b200._lib import load_library  # noqa: E402

lib = load_library()
names = ["select+dots+warp reduce", "smem + barrier", "cta sum + push", "mbarrier wait",
         "cluster totals+barrier", "scalars", "update"]
rng = np.random.default_rng(0)
for (m, k) in [(200, 32), (500, 32), (1000, 32), (2000, 32), (4000, 32)]:
    B = rng.standard_normal((m, k))
    for rep in range(2):
        K.qr_house(B)
    buf = np.zeros(32 * 8, np.int64)
    lib.spq_debug_panel_trace(buf.ctypes.data_as(C.POINTER(C.c_longlong)), buf.size)
    t = buf.reshape(32, 8)
    per = np.diff(t[2:30, 0])
    d = np.diff(t[2:30], axis=1)
    print(f"m={m}: cycles/column {per.mean():.0f} ({per.mean() / 1.965e3:.2f} us)")
    for i, nm in enumerate(names):
        print(f"   {nm:26s} {d[:, i].mean():8.0f}")
