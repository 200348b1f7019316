"""C3 device timeline: SPQ_SCOPE_LOG must be set; factorizes 3x with marks and
collects timings after each (the scope log gets family, ms, start-offset, tag).
Diagnostic only."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_06807_b200.factor import factorize  # noqa: E402
from paper_2010_06807_b200.ordering import partition_geometric  # noqa: E402
from paper_2010_06807_b200.problems import make_config  # noqa: E402

A, dims, L, eps, b, tol = make_config(sys.argv[1] if len(sys.argv) > 1 else "C3")
tree = partition_geometric(dims, L)
for r in range(3):
    t0 = time.perf_counter()
    F = factorize(A, tree, eps=eps, _marks=True)
    t1 = time.perf_counter()
    tm = F.device_timings()
    log = os.environ.get("SPQ_SCOPE_LOG")
    if log:
        with open(log, "a") as f:
            f.write(f"# factorization {r} wall {1e3 * (t1 - t0):.2f} ms device {F.device_ms:.2f} ms\n")
    print(r, round(1e3 * (t1 - t0), 2), round(F.device_ms, 2), tm["host"], flush=True)
    del F
