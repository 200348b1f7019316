"""Per-kernel device timings through the plugin API (QR panels, larft)."""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2010_06807_b200 import kernels as K  # noqa: E402

ctx = K._context()
out = {}
rng = np.random.default_rng(0)
for (m, k) in [(124, 84), (4000, 125), (10000, 200), (2000, 820), (1313, 1313)]:
    B = rng.standard_normal((m, k))
    K.qr_house(B)                       # warm
    ctx.call("spq_reset_timings")
    panel, R = K.qr_house(B)
    t = ctx.timings()
    out[f"qr_{m}x{k}"] = {f: round(t[f]["ms"], 3) for f in ("qr", "wy", "copy") if t[f]["ms"]}
for k in (128, 820, 1313):
    V = np.tril(rng.standard_normal((k + 50, k)), -1) + np.eye(k + 50, k)
    tau = rng.uniform(1, 2, k)
    ctx.call("spq_reset_timings")
    K.build_t(V, tau)
    t = ctx.timings()
    out[f"build_t_{k}"] = {f: round(t[f]["ms"], 3) for f in ("qr", "wy") if t[f]["ms"]}
print(json.dumps(out, indent=1))
