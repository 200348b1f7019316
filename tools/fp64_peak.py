"""Measure the fp64 roofline denominators on the box: cuBLAS DGEMM (torch),
our DMMA GEMM at the WY shapes, and a device copy bandwidth."""
import ctypes as C
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2010_06807_b200._lib import Context  # noqa: E402


def cublas_dgemm(n=8192, reps=10):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return 2.0 * n ** 3 / (best * 1e-3) / 1e12


out = {"cublas_dgemm_tflops_8192": cublas_dgemm()}
ctx = Context()
ms = C.c_float()
for (m, n, k, ta) in [(4096, 4096, 4096, 0), (3500, 3700, 122, 0), (122, 3700, 3500, 1),
                      (8192, 8192, 256, 0), (128, 8192, 8192, 1)]:
    ctx.call("spq_bench_gemm", m, n, k, ta, 10, C.byref(ms))
    out[f"dmma_{m}x{n}x{k}_tA{ta}_tflops"] = 2.0 * m * n * k / (ms.value * 1e-3) / 1e12
print(json.dumps(out, indent=1))
