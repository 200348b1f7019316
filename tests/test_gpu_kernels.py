"""Per-kernel parity of the sm_100a plugin API against the reference's
known-answer vectors (tests/golden/kernels.npz, produced by the reference's
numba backend) and the reference test suite's closed-form cases
(`pkg/tests/test_kernels.py`)."""

import numpy as np
import pytest

from parity import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def K():
    from paper_2010_06807_b200 import kernels
    return kernels


@pytest.fixture(scope="module")
def gk():
    return dict(np.load(f"{GOLDEN}/kernels.npz"))


def test_qr_house_golden(K, gk):
    for t in range(int(gk["n_qr"])):
        B = gk[f"qr{t}_B"]
        panel, R = K.qr_house(B)
        Rr = gk[f"qr{t}_R"]
        sc = max(np.abs(Rr).max(), 1.0)
        assert np.abs(R - Rr).max() <= 1e-12 * sc, t
        assert np.abs(panel.tau - gk[f"qr{t}_tau"]).max() <= 1e-12, t
        assert np.abs(panel.V - gk[f"qr{t}_V"]).max() <= 1e-10, t
        assert np.abs(panel.T - gk[f"qr{t}_T"]).max() <= 1e-10 * max(1, np.abs(gk[f"qr{t}_T"]).max()), t
        HtC = K.apply_panel_left(panel, gk[f"qr{t}_C"], transpose=True)
        assert np.abs(HtC - gk[f"qr{t}_HtC"]).max() <= 1e-11 * max(1, np.abs(HtC).max()), t
        assert (np.diag(R) >= 0).all()


def test_qr_closed_forms(K):
    panel, R = K.qr_house(np.array([[3.0], [4.0]]))
    assert abs(R[0, 0] - 5.0) <= 1e-14
    out = panel.apply(np.array([3.0, 4.0]), transpose=True)
    assert np.allclose(out, [5.0, 0.0], atol=1e-14)
    panel, R = K.qr_house(np.eye(3))
    assert np.allclose(R, np.eye(3), atol=1e-15)
    panel, R = K.qr_house(np.zeros((4, 1)))
    assert panel.tau[0] == 0.0 and R[0, 0] == 0.0
    from paper_2010_06807_b200.errors import NestqrError
    with pytest.raises(NestqrError):
        K.qr_house(np.ones((2, 3)))


@pytest.mark.parametrize("m,k", [(32, 8), (128, 64), (512, 96), (1500, 130), (3000, 300)])
def test_qr_orthogonality_and_reconstruction(K, m, k):
    rng = np.random.default_rng(m + k)
    B = rng.standard_normal((m, k))
    panel, R = K.qr_house(B)
    Q = panel.apply(np.eye(m))
    assert np.linalg.norm(Q.T @ Q - np.eye(m)) <= 1e-12 * k
    S = np.vstack([R, np.zeros((m - k, k))])
    assert np.linalg.norm(panel.apply(S) - B) <= 1e-13 * np.linalg.norm(B) * max(1, k / 32)
    _, Rref = np.linalg.qr(B)
    s = np.sign(np.diag(Rref))
    assert np.abs(s[:, None] * Rref - R).max() <= 1e-11 * np.abs(R).max()


def test_rrqr_golden(K, gk):
    for key in gk["rr_keys"]:
        t = key.split("_")[0]
        M = gk[f"{t}_M"]
        eps = float(gk[key + "_eps"])
        res = K.rrqr_threshold(M, eps)
        assert res.rank == int(gk[key + "_rank"]), key
        Rr = gk[key + "_R"]
        r = res.rank
        # steps whose pivot column is pure rounding noise (|R_ii| <= 1e-11 |R_00|,
        # e.g. eps = 0 on a rank-deficient M) pick arbitrary pivots in any
        # implementation, the reference's two backends included
        d = np.abs(np.diag(Rr[:, :r])) if r else np.zeros(0)
        sig = int(np.sum(d > 1e-11 * d[0])) if r else 0
        assert np.array_equal(res.perm[:sig], gk[key + "_perm"][:sig]), key
        assert np.abs(res.R[:sig, :sig] - Rr[:sig, :sig]).max(initial=0) <= 1e-10 * max(1, np.abs(Rr).max()), key
        # tau of steps on tiny (sigma ~ 1e-8) columns is rounding-sensitive; R pins them
        assert np.abs(res.panel.tau[:sig] - gk[key + "_tau"][:sig]).max(initial=0) <= 1e-8, key


def test_rrqr_properties(K):
    assert K.rrqr_threshold(np.zeros((4, 6)), 1e-3).rank == 0
    assert K.rrqr_threshold(np.eye(3), 0.5).rank == 3
    rng = np.random.default_rng(8)
    M = rng.standard_normal((12, 9))
    res = K.rrqr_threshold(M, 1e-8)
    S = np.zeros((12, 9))
    S[:res.rank] = res.R
    S[res.rank:, res.rank:] = res.resid
    assert np.allclose(res.q_dense() @ S, M[:, res.perm], atol=1e-12)
    Mo = np.outer(rng.standard_normal(8), rng.standard_normal(8))
    assert K.rrqr_threshold(Mo, 1e-6).rank == 1
    assert K.rrqr_threshold(Mo, 1e-6, min_rank=3).rank >= 3


def test_tri_solve_golden(K, gk):
    for t in range(int(gk["n_ts"])):
        R = gk[f"ts{t}_R"]
        X = K.tri_solve(R, gk[f"ts{t}_C"], side="left")
        assert np.abs(X - gk[f"ts{t}_left"]).max() <= 1e-12 * max(1, np.abs(X).max())
        Y = K.tri_solve(R, gk[f"ts{t}_Cr"], side="right")
        assert np.abs(Y - gk[f"ts{t}_right"]).max() <= 1e-12 * max(1, np.abs(Y).max())


def test_tri_solve_singular(K):
    from paper_2010_06807_b200.errors import SingularPivotError
    R = np.diag([2.0, 1e-20, 1.0])
    with pytest.raises(SingularPivotError) as e:
        K.tri_solve(R, np.ones(3))
    assert e.value.index == 1
    with pytest.raises(SingularPivotError) as e:
        K.tri_solve(np.diag([0.0, 1.0]), np.ones(2))
    assert e.value.index == 0


def test_build_t_matches_golden(K, gk):
    for t in range(int(gk["n_qr"])):
        T = K.build_t(gk[f"qr{t}_V"], gk[f"qr{t}_tau"])
        Tr = gk[f"qr{t}_T"]
        assert np.abs(T - Tr).max() <= 1e-11 * max(1, np.abs(Tr).max())


def test_nestqr_backend_module_contract(golden_dir):
    """The `nestqr.kernels._impl` drop-in (paper_2010_06807_b200.nestqr_backend)
    returns what the reference's numba backend returned on the golden inputs:
    house_qr's (V, tau, R), build_t's T, cpqr_threshold's (V, tau, perm, r)
    and both triangular solves."""
    import os
    from paper_2010_06807_b200 import nestqr_backend as NB
    g = dict(np.load(os.path.join(golden_dir, "kernels.npz")))
    for t in range(int(g["n_qr"])):
        V, tau, R = NB.house_qr(g[f"qr{t}_B"])
        sc = max(1.0, np.abs(g[f"qr{t}_R"]).max())
        assert np.abs(R - g[f"qr{t}_R"]).max() <= 1e-12 * sc
        assert np.abs(tau - g[f"qr{t}_tau"]).max() <= 1e-12
        assert np.abs(V - g[f"qr{t}_V"]).max() <= 1e-10
        T = NB.build_t(V, tau)
        assert np.abs(T - g[f"qr{t}_T"]).max() <= 1e-10 * max(1.0, np.abs(T).max())
    for key in g["rr_keys"]:
        t = key.split("_")[0]
        V, tau, Tred, perm, r = NB.cpqr_threshold(g[f"{t}_M"], float(g[key + "_eps"]), 0)
        assert r == int(g[key + "_rank"]), key
        assert V.shape[1] == r and tau.shape == (r,) and perm.dtype == np.int64
    for t in range(int(g["n_ts"])):
        R = g[f"ts{t}_R"]
        X = NB.tri_solve_left(R, g[f"ts{t}_C"])
        assert np.abs(X - g[f"ts{t}_left"]).max() <= 1e-12 * max(1.0, np.abs(X).max())
        Y = NB.tri_solve_right(R, g[f"ts{t}_Cr"])
        assert np.abs(Y - g[f"ts{t}_right"]).max() <= 1e-12 * max(1.0, np.abs(Y).max())
