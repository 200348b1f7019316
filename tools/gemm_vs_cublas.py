"""Our DMMA GEMM vs cuBLAS DGEMM (torch.matmul) at the compact-WY shapes of the
C3 / C4 / C5 fronts: headroom of the WY family. Diagnostic."""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2010_06807_b200._lib import Context  # noqa: E402


def cublas(m, n, k, ta, reps=10):
    a = torch.randn(k, m, dtype=torch.float64, device="cuda") if ta else \
        torch.randn(m, k, dtype=torch.float64, device="cuda")
    b = torch.randn(k, n, dtype=torch.float64, device="cuda")
    op = (lambda: torch.matmul(a.t(), b)) if ta else (lambda: torch.matmul(a, b))
    op()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        op()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return 2.0 * m * n * k / (best * 1e-3) / 1e12


ctx = Context()
ms = C.c_float()
rows = []
for (m, n, k, ta) in [(4015, 3985, 104, 0), (104, 3985, 4015, 1), (2000, 2500, 60, 0), (60, 2500, 2000, 1),
                      (120, 120, 2000, 1), (8000, 8000, 400, 0), (400, 8000, 8000, 1),
                      (16900, 15400, 1790, 0), (1790, 15400, 16900, 1), (4096, 4096, 4096, 0)]:
    ctx.call("spq_bench_gemm", m, n, k, ta, 10, C.byref(ms))
    ours = 2.0 * m * n * k / (ms.value * 1e-3) / 1e12
    ref = cublas(m, n, k, ta)
    rows.append({"m": m, "n": n, "k": k, "transA": ta, "ours_tflops": round(ours, 2),
                 "cublas_tflops": round(ref, 2), "ratio": round(ours / ref, 2)})
    print(rows[-1], flush=True)
json.dump(rows, open(sys.argv[1], "w"), indent=1) if len(sys.argv) > 1 else None
