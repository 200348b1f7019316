"""Python-side profile of the public factorize() call at C3 (what the bench's e2e
number adds on top of the device span). Diagnostic only."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from paper_2010_06807_b200 import factor as FZ  # noqa: E402
from paper_2010_06807_b200.ordering import partition_geometric  # noqa: E402
from paper_2010_06807_b200.problems import make_config  # noqa: E402

A, dims, L, eps, b, tol = make_config("C3")
tree = partition_geometric(dims, L)
for _ in range(3):
    F = FZ.factorize(A, tree, eps=eps, device=0)
    del F
torch.cuda.synchronize()
pr = cProfile.Profile()
for _ in range(3):
    t0 = time.perf_counter()
    pr.enable()
    F = FZ.factorize(A, tree, eps=eps, device=0, _marks=True)
    pr.disable()
    torch.cuda.synchronize()
    print("wall ms", round(1e3 * (time.perf_counter() - t0), 2), "device ms", round(F.device_ms, 2), flush=True)
    del F
pstats.Stats(pr).sort_stats("cumulative").print_stats(35)
pstats.Stats(pr).sort_stats("tottime").print_stats(20)
