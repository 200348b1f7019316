"""Compare GPU sparsification ranks at n=48 (C5 generator) with an oracle run
(stop_level=8) saved to tools/_oracle48_ranks.npy [(lev, p, rank, before)]."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_2010_06807_b200.problems import make_config
from paper_2010_06807_b200.ordering import partition_geometric
from paper_2010_06807_b200.factor import factorize

A, dims, L, eps, b, tol = make_config("C5", n=48)
tree = partition_geometric(dims, L)
t = time.time()
F = factorize(A, tree, eps=eps)
print("factor", time.time() - t)
o = np.load("tools/_oracle48_ranks.npy")
ref = {(int(l), int(p)): (int(r), int(bf)) for l, p, r, bf in o}
got = {(int(l), int(p)): (int(r), int(bf)) for l, p, bf, r in F.sparsify_log}
same = diff = missing = 0
for k, v in sorted(ref.items(), reverse=True):
    if k not in got:
        missing += 1
        continue
    if got[k] == v:
        same += 1
    else:
        diff += 1
        if diff <= 20:
            print("diff", k, "oracle (rank,before)", v, "gpu", got[k])
print("levels>=8: same", same, "diff", diff, "missing", missing)
