"""Device-side view of the occasional slow step: per factorization the
longest timed scopes (SPQ_SCOPE_LOG must be set). Diagnostic."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2010_06807_b200.factor import factorize  # noqa: E402
from paper_2010_06807_b200.ordering import partition_geometric  # noqa: E402
from paper_2010_06807_b200.problems import make_config  # noqa: E402

log = os.environ["SPQ_SCOPE_LOG"]
A, dims, L, eps, b, tol = make_config("C3")
tree = partition_geometric(dims, L)
pos = 0
for r in range(45):
    t0 = time.perf_counter()
    F = factorize(A, tree, eps=eps, _marks=True)
    wall = time.perf_counter() - t0
    F.device_timings()
    del F
    lines = open(log).read().splitlines()
    new, pos = lines[pos:], len(lines)
    rows = []
    for l in new:
        p = l.split(" ", 3)
        try:
            rows.append((float(p[1]), int(p[0]), float(p[2]), p[3] if len(p) > 3 else ""))
        except (ValueError, IndexError):
            pass
    rows.sort(reverse=True)
    flag = "SLOW" if wall > 0.16 else ""
    print(f"{r} wall {1e3 * wall:.1f} ms {flag} top scopes: " +
          " | ".join(f"fam{f} {d:.2f}ms @{s:.1f} {t[:70]}" for d, f, s, t in rows[:3]), flush=True)
