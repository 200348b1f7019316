"""Host-side logic on CPU: ordering restatement pinned to the reference's
trees, generator properties, host GMRES, C-ABI symbol export, and the
multi-process (replica) bench path under gloo."""

import json
import os
import re

import numpy as np
import pytest

from parity import GOLDEN

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("case", ["C1", "C3", "C4", "C1_n24", "C3_n48", "C4_n12", "odd", "odd3"])
def test_tree_matches_reference_digest(case):
    from paper_2010_06807_b200.ordering import partition_geometric, tree_digest
    d = json.load(open(os.path.join(GOLDEN, "trees.json")))[case]
    assert tree_digest(partition_geometric(tuple(d["dims"]), d["L"])) == d["sha256"]


def test_upwind_generator_structure():
    from paper_2010_06807_b200.problems import UpwindSpec, upwind_convection_diffusion
    A = upwind_convection_diffusion(UpwindSpec(n=6, ndim=2, beta_const=(20.0, 20.0)))
    D = A.to_dense()
    h = 1 / 7
    # interior node, beta > 0: west/south couplings carry -beta/h extra
    i = 2 * 6 + 3
    assert np.isclose(D[i, i - 1], -1 / h ** 2 - 20 / h)
    assert np.isclose(D[i, i + 1], -1 / h ** 2)
    assert np.isclose(D[i, i - 6], -1 / h ** 2 - 20 / h)
    assert np.isclose(D[i, i], 4 / h ** 2 + 40 / h)
    # pattern symmetric, values not
    assert ((D != 0) == (D.T != 0)).all() and not np.allclose(D, D.T)
    # column-diagonal dominance of the upwind M-matrix
    assert (np.diag(D) > 0).all()


def test_generator_seeded_and_variable():
    from paper_2010_06807_b200.problems import make_config
    A1 = make_config("C3", n=20)[0]
    A2 = make_config("C3", n=20)[0]
    assert np.array_equal(A1.data, A2.data)
    A4 = make_config("C4", n=6)[0]
    assert A4.ncols == 216 and A4.nnz == 216 + 6 * 5 * 36


def test_host_gmres_with_oracle():
    """The host GMRES restatement (test comparator for spq_gmres) solves the
    oracle-preconditioned system to the dense solution."""
    from oracle import spaqr_oracle as O
    from oracle.krylov import gmres_host
    from paper_2010_06807_b200.ordering import partition_geometric
    from paper_2010_06807_b200.problems import make_config
    from paper_2010_06807_b200.sparse import matvec
    A, dims, L, eps, b, tol = make_config("C1", n=20)
    F = O.factorize(A, partition_geometric(dims, L), eps=1e-2)
    x, its, hist, conv = gmres_host(A, b, F, tol=1e-12, maxit=50, matvec=matvec)
    assert conv
    xd = np.linalg.solve(A.to_dense(), b)
    assert np.linalg.norm(x - xd) <= 1e-9 * np.linalg.norm(xd)
    x0, its0, _, _ = gmres_host(A, np.zeros_like(b), F, matvec=matvec)
    assert its0 == 0 and not x0.any()


def test_product_gmres_needs_device_or_reference():
    """No silent host fallback in the product package: a non-B200 F goes to
    the reference's own nestqr.solve.gmres or raises."""
    import importlib.util
    from oracle import spaqr_oracle as O
    from paper_2010_06807_b200.errors import NestqrError
    from paper_2010_06807_b200.ordering import partition_geometric
    from paper_2010_06807_b200.problems import make_config
    from paper_2010_06807_b200.solve import gmres
    A, dims, L, eps, b, tol = make_config("C1", n=12)
    F = O.factorize(A, partition_geometric(dims, L), eps=1e-2)
    if importlib.util.find_spec("nestqr") is None:
        with pytest.raises(NestqrError):
            gmres(A, b, F)
    else:
        x, rep = gmres(A, b, F)
        assert rep.converged


def test_library_exports_every_header_symbol():
    from paper_2010_06807_b200._lib import SIGNATURES, load_library
    lib = load_library()
    hdr = open(os.path.join(ROOT, "include", "spaqr_b200.h")).read()
    names = set(re.findall(r"\b(spq_[a-z_0-9]+)\s*\(", hdr))
    assert names == set(SIGNATURES)
    for n in names:
        assert hasattr(lib, n), n


def test_no_silent_cpu_fallback():
    """Without an sm_100a device the product path must fail loudly."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2010_06807_b200.errors import NestqrError
    from paper_2010_06807_b200.factor import factorize
    from paper_2010_06807_b200.ordering import partition_geometric
    from paper_2010_06807_b200.problems import make_config
    A, dims, L, eps, b, tol = make_config("C1", n=16)
    with pytest.raises(NestqrError):
        factorize(A, partition_geometric(dims, 3), eps=eps)


def _replica_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, ROOT)
    from bench import reduce_max
    from oracle import spaqr_oracle as O
    from paper_2010_06807_b200.ordering import partition_geometric
    from paper_2010_06807_b200.problems import make_config
    A, dims, L, eps, b, tol = make_config("C1", n=16)
    import time
    t0 = time.perf_counter()
    F = O.factorize(A, partition_geometric(dims, L), eps=eps)
    dt = (time.perf_counter() - t0) * 1e3 + 100.0 * rank
    T = reduce_max([dt, 2 * dt], dist, device="cpu")
    q.put((rank, T, int(F.ranks[0][2]) if F.ranks else -1))
    dist.destroy_process_group()


def test_replica_timing_is_max_over_ranks_gloo():
    import multiprocessing as mp
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_replica_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    Ts = [o[1] for o in out]
    assert Ts[0] == Ts[1]            # every rank sees the max
    assert Ts[0][0] >= 100.0         # rank 1's (shifted) time wins
    assert out[0][2] == out[1][2]    # replicas compute identical ranks


def test_bench_gpus_flag_spawns_ranks():
    """`bench.py --gpus 2` with no launcher re-executes itself under torchrun:
    two ranks, one JSON line from rank 0 (reference arm, gloo, C1)."""
    import subprocess
    import sys
    env = dict(os.environ, SPQ_BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--gpus", "2", "--config", "C1", "--steps", "1", "--warmup", "0"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1
    assert lines[0]["n_gpus"] == 2 and lines[0]["impl"] == "reference"
    assert lines[0]["config"]["config"] == "C1" and lines[0]["config"]["N"] == 4096


@pytest.mark.parametrize("cfg,n", [("C1", 24), ("C3", 48), ("C4", 12)])
def test_symbolic_fill_levels_match_reference(cfg, n):
    """The symbolic (drop-free) fill prediction equals the live reference's
    `symbolic_fill_levels` (factor.py:1004-1050) level by level (golden
    written by tests/golden/make_symbolic.py)."""
    from paper_2010_06807_b200.ordering import partition_geometric
    from paper_2010_06807_b200.problems import make_config
    from paper_2010_06807_b200.symbolic import symbolic_fill_levels
    g = np.load(os.path.join(GOLDEN, "symbolic.npz"))
    A, dims, L, eps, b, tol = make_config(cfg, n=n)
    tree = partition_geometric(dims, L)
    pat = symbolic_fill_levels(A, tree)
    assert sorted(pat) == list(range(1, L + 1))
    for lev, pairs in pat.items():
        ref = {tuple(p) for p in g[f"{cfg}_n{n}_L{lev}"].tolist()}
        assert pairs == ref, (lev, len(pairs), len(ref))
