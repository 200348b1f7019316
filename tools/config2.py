"""BASELINE config 2 on the B200: batched QR + Q^T-apply (4096 blocks) and
batched threshold RRQR (4096 x 64x192 at 1e-2, 1e-4).  Prints one JSON line
with device GFLOP/s (LAPACK-standard counts) and the ranks."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2010_06807_b200.batched import batched_qr, batched_rrqr, config2_inputs  # noqa: E402

t0 = time.perf_counter()
Bs, Cs, Ms = config2_inputs()
gen = time.perf_counter() - t0
out = {"gen_s": gen}
fl_qr = sum(2 * b.shape[0] * b.shape[1] ** 2 - 2 * b.shape[1] ** 3 / 3 for b in Bs)
fl_ap = sum(4 * b.shape[0] * c.shape[1] * b.shape[1] - c.shape[1] * b.shape[1] ** 2
            for b, c in zip(Bs, Cs))
best = 1e9
for _ in range(3):
    Rs, Co, ms = batched_qr(Bs, Cs)
    best = min(best, ms)
out["qr_apply_ms"] = best
out["qr_apply_gflops"] = (fl_qr + fl_ap) / (best * 1e-3) / 1e9
for eps in (1e-2, 1e-4):
    best = 1e9
    for _ in range(3):
        ranks, rd, ms = batched_rrqr(Ms, eps)
        best = min(best, ms)
    m, n = 64, 192
    fl = sum(4 * m * n * r - 2 * r * r * (m + n) + 4 * r ** 3 / 3 for r in ranks)
    out[f"rrqr_{eps:g}_ms"] = best
    out[f"rrqr_{eps:g}_gflops"] = fl / (best * 1e-3) / 1e9
    out[f"rrqr_{eps:g}_ranks"] = [int(ranks.min()), int(np.median(ranks)), int(ranks.max())]
print(json.dumps(out))
