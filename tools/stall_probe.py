"""Which C-ABI call carries the occasional +85 ms step?  Times every library
call of 60 C3 factorizations and prints, for the slow steps, the calls that
took unusually long.  Diagnostic."""
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2010_06807_b200._lib as L  # noqa: E402
from paper_2010_06807_b200.factor import factorize  # noqa: E402
from paper_2010_06807_b200.ordering import partition_geometric  # noqa: E402
from paper_2010_06807_b200.problems import make_config  # noqa: E402

log = []
orig = L.Context.call


def timed(self, name, *a):
    t0 = time.perf_counter()
    try:
        return orig(self, name, *a)
    finally:
        log.append((name, time.perf_counter() - t0, time.perf_counter()))


L.Context.call = timed
A, dims, Lv, eps, b, tol = make_config("C3")
tree = partition_geometric(dims, Lv)
for _ in range(3):
    factorize(A, tree, eps=eps)
steps = []
for s in range(60):
    log.clear()
    t0 = time.perf_counter()
    F = factorize(A, tree, eps=eps)
    F._ctx.call("spq_synchronize")
    dt = time.perf_counter() - t0
    steps.append((dt, list(log)))
    del F
med = np.median([d for d, _ in steps])
base = collections.defaultdict(list)
for d, lg in steps:
    if d < 1.1 * med:
        for i, (n, t, _) in enumerate(lg):
            base[(i, n)].append(t)
print(f"median step {1e3 * med:.1f} ms; steps: " + " ".join(f"{1e3 * d:.0f}" for d, _ in steps))
for k, (d, lg) in enumerate(steps):
    if d > 1.25 * med:
        print(f"slow step {k}: {1e3 * d:.1f} ms")
        for i, (n, t, _) in enumerate(lg):
            ref = np.median(base.get((i, n), [0.0]))
            if t - ref > 0.01:
                print(f"   call #{i} {n}: {1e3 * t:.1f} ms (typical {1e3 * ref:.1f})")
        tot = sum(t for _, t, _ in lg)
        print(f"   in-library {1e3 * tot:.1f} ms of {1e3 * d:.1f}")
print("typical per-call wall (ms), calls in order:")
order = sorted(base, key=lambda k: k[0])
for i, n in order:
    t = 1e3 * float(np.median(base[(i, n)]))
    if t >= 0.3:
        print(f"   #{i:3d} {n:28s} {t:7.2f}")
print(f"sum of medians {1e3 * sum(float(np.median(v)) for v in base.values()):.1f} ms")
