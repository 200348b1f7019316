"""GPU parity of the full factorization path against the reference's golden
vectors (tests/golden, generated from the live reference) and against the
CPU oracle on the same seeded inputs."""

import numpy as np
import pytest

from parity import (compare_chains, compare_records, compare_structure, load, payload_ok,
                    rss_bar, rss_diag_errors)

pytestmark = pytest.mark.gpu


def _views(F):
    from paper_2010_06807_b200.factor import BlockHouseholder, InterfaceScaling, Sparsifier
    q = F.q_chain
    return ([r for r in q if isinstance(r, BlockHouseholder)],
            [r for r in q if isinstance(r, InterfaceScaling)],
            [r for r in q if isinstance(r, Sparsifier)])


def _check_against_reference(F, rep, g):
    """Everything the golden holds: structure, ranks, R_ss / R_sn / R_pp /
    sparsifier bases per record, the chains, GMRES."""
    problems = compare_structure(F.stats, F.sparsify_log, F.row_of_col, g)
    assert not problems, "\n".join(problems[:20])
    problems = compare_records(*_views(F), g)
    assert not problems, "\n".join(problems[:20])
    problems = compare_chains(F, g)
    assert not problems, "\n".join(problems)
    assert payload_ok(F.payload_scalars, g), (F.payload_scalars, int(g["payload"]))
    gi, gres = int(g["gmres_iters"]), float(g["gmres_hist"][-1])
    assert abs(rep.iterations - gi) <= 1
    assert rep.final_residual <= 10 * max(gres, 1e-16) and rep.converged


def _run(name, cfg, n, **opts):
    from paper_2010_06807_b200.factor import factorize
    from paper_2010_06807_b200.ordering import partition_geometric
    from paper_2010_06807_b200.problems import make_config
    from paper_2010_06807_b200.solve import gmres
    A, dims, L, eps, b, tol = make_config(cfg, n=n)
    tree = partition_geometric(dims, L)
    F = factorize(A, tree, eps=eps, **opts)
    x, rep = gmres(A, b, F, tol=tol)
    return A, b, F, x, rep


@pytest.mark.parametrize("name,cfg,n", [("C1_n24", "C1", 24), ("C3_n48", "C3", 48),
                                        ("C4_n12", "C4", 12), ("C1", "C1", None)])
def test_factor_matches_reference(name, cfg, n):
    g = load(name)
    A, b, F, x, rep = _run(name, cfg, n)
    _check_against_reference(F, rep, g)


@pytest.mark.parametrize("name,cfg,n,opts", [
    ("C1_unscaled", "C1", None, {"mode": "unscaled"}),
    ("C3_n48_unscaled", "C3", 48, {"mode": "unscaled"}),
    ("C4_n12_unscaled", "C4", 12, {"mode": "unscaled"}),
    ("C3_n96_unscaled", "C3", 96, {"mode": "unscaled"}),
    ("C1_se2", "C1", None, {"scale_every": 2}),
    ("C3_n48_se2", "C3", 48, {"scale_every": 2}),
    ("C3_n96_se2", "C3", 96, {"scale_every": 2}),
])
def test_unscaled_route_matches_reference(name, cfg, n, opts):
    """§8(f) row 3: the unscaled sparsification route (sigma-weighted target,
    H_f elimination of the fine columns, R_ff / R_fc records, min_rank
    escalation; factor.py:557-566, 660-709), alone (mode='unscaled') and
    alternating with scaled levels (scale_every=2), against the live
    reference's goldens: ranks, stats, dropped_max, R_ff / R_fc / H_f, every
    R_ss / R_sn / R_pp, the chains and GMRES."""
    g = load(name)
    A, b, F, x, rep = _run(name, cfg, n, **opts)
    _check_against_reference(F, rep, g)


def test_chains_match_oracle():
    """apply_qt / solve_w / apply_w on the device equal the CPU oracle's
    chains on the same factorization input (C3 shape at 40^2)."""
    from oracle import spaqr_oracle as O
    from paper_2010_06807_b200.factor import factorize
    from paper_2010_06807_b200.ordering import partition_geometric
    from paper_2010_06807_b200.problems import make_config
    A, dims, L, eps, b, tol = make_config("C3", n=40)
    tree = partition_geometric(dims, L)
    F = factorize(A, tree, eps=eps)
    Fo = O.factorize(A, tree, eps=eps)
    rng = np.random.default_rng(5)
    for nrhs in (1, 3):
        v = rng.standard_normal((A.ncols, nrhs)) if nrhs > 1 else rng.standard_normal(A.ncols)
        for fn in ("apply_qt", "solve_w", "apply_w"):
            a = getattr(F, fn)(v)
            o = getattr(Fo, fn)(v)
            assert np.abs(a - o).max() <= 1e-8 * max(np.abs(o).max(), 1.0), fn


@pytest.mark.parametrize("opts", [{}, {"mode": "unscaled"}])
def test_split_back_substitution(monkeypatch, opts):
    """Large R_ss are split into row blocks at chain compile time (one op per
    block, the products with the solved part spread over CTAs); forced here
    at 32 rows so every separator of a small problem takes that route, with
    multiple right-hand sides, against the unsplit device chains and (scaled
    mode) the CPU oracle's."""
    from oracle import spaqr_oracle as O
    from paper_2010_06807_b200.factor import factorize
    from paper_2010_06807_b200.ordering import partition_geometric
    from paper_2010_06807_b200.problems import make_config
    A, dims, L, eps, b, tol = make_config("C3", n=48)
    tree = partition_geometric(dims, L)
    rng = np.random.default_rng(11)
    vs = [rng.standard_normal(A.ncols), rng.standard_normal((A.ncols, 2))]
    fns = ("solve_w", "apply_w", "apply_qt")

    def run(split):
        if split:
            monkeypatch.setenv("SPQ_CHAIN_SPLIT_K", "32")
        else:
            monkeypatch.delenv("SPQ_CHAIN_SPLIT_K", raising=False)
        F = factorize(A, tree, eps=eps, **opts)
        out = [getattr(F, fn)(v) for v in vs for fn in fns]   # chains compile at first use
        info = np.zeros(4, np.int64)
        F._ctx.call("spq_chain_info", 1, info)
        return out, int(info[1])

    split, nsplit = run(True)
    whole, nwhole = run(False)
    assert nsplit > nwhole            # the separators' back substitutions became several ops
    for a, o in zip(split, whole):
        assert np.abs(a - o).max() <= 1e-10 * max(np.abs(o).max(), 1.0)
    if not opts:
        Fo = O.factorize(A, tree, eps=eps)
        ref = [getattr(Fo, fn)(v) for v in vs for fn in fns]
        for a, o in zip(split, ref):
            assert np.abs(a - o).max() <= 1e-8 * max(np.abs(o).max(), 1.0)


def test_exact_mode_identity():
    """eps = 0 / no sparsification: P^T Q^T A W^{-1} = I (reference
    test_factor.py:395-402) and W^T W = A^T A for the equilibrated A."""
    from paper_2010_06807_b200.factor import factorize
    from paper_2010_06807_b200.ordering import partition_geometric
    from paper_2010_06807_b200.problems import make_config
    for sparsify in (False, True):
        A, dims, L, eps, b, tol = make_config("C1", n=16)
        tree = partition_geometric(dims, 3)
        F = factorize(A, tree, eps=0.0, sparsify=sparsify)
        M = F.materialize_preconditioned()
        assert np.linalg.norm(M - np.eye(A.ncols)) <= 1e-11
        W = F.materialize_w()
        D = A.to_dense()
        assert np.linalg.norm(W.T @ W - D.T @ D) <= 1e-10 * np.linalg.norm(D.T @ D)
        Y = np.random.default_rng(0).standard_normal(A.ncols)
        assert np.allclose(F.apply_w(F.solve_w(Y)), Y, atol=1e-11)


def test_singular_pivot_raises():
    from paper_2010_06807_b200.errors import SingularPivotError
    from paper_2010_06807_b200.factor import factorize
    from paper_2010_06807_b200.ordering import partition_geometric
    from paper_2010_06807_b200.sparse import SparseMat
    n = 8
    D = np.eye(n * n)
    D[3, 3] = 0.0          # empty column -> zero pivot in its leaf block
    A = SparseMat.from_dense(D)
    tree = partition_geometric((n, n), 2)
    with pytest.raises(SingularPivotError):
        factorize(A, tree, eps=0.0, sparsify=False, equilibrate=False)


@pytest.mark.slow
def test_c3_full_matches_reference():
    """BASELINE metric config (256^2, L=10, eps=1e-3) against the reference's
    golden run: identical per-interface ranks and statistics; R_ss, R_sn,
    R_pp and the sparsifier bases of every record and the reference's own
    chain outputs within 10x the reference's numba-vs-numpy envelope;
    GMRES its +-1."""
    g = load("C3")
    A, b, F, x, rep = _run("C3", "C3", None)
    _check_against_reference(F, rep, g)


@pytest.mark.slow
def test_c4_full_matches_reference():
    """BASELINE config 4 (3D 32^3, L=9, eps=1e-2; the reference needs ~210 s
    on the CPU) against its golden run, same comparisons as C3."""
    g = load("C4")
    A, b, F, x, rep = _run("C4", "C4", None)
    _check_against_reference(F, rep, g)


@pytest.mark.slow
def test_c5_full_size_properties():
    """BASELINE config 5 (3D 64^3, N=262,144, L=11): the CPU oracle cannot run
    it (the reference OOMs at 62 GB), so parity rests on
    size-independent properties: GMRES reaches the config's 1e-10 true
    residual, W^-1 W = I and Q^T is an isometry on random vectors."""
    import gc
    gc.collect()   # earlier tests' contexts: C5 needs most of the 180 GB
    A, b, F, x, rep = _run("C5", "C5", None)
    assert rep.converged and rep.final_residual <= 1e-10
    rng = np.random.default_rng(7)
    y = rng.standard_normal(A.ncols)
    assert np.linalg.norm(F.apply_w(F.solve_w(y)) - y) <= 1e-8 * np.linalg.norm(y)
    z = F.apply_qt(y)
    assert abs(np.linalg.norm(z) - np.linalg.norm(y)) <= 1e-10 * np.linalg.norm(y)


@pytest.mark.slow
def test_n48_3d_top_levels_match_oracle(golden_dir):
    """3D 48^3 with the C5 generator: every sparsified interface on levels
    11..8 has the oracle's rank (tests/golden/make_n48_ranks.py).  Level 8
    has candidate matrices with > 65,535 columns (grid-limit regression)."""
    import os
    from paper_2010_06807_b200.factor import factorize
    from paper_2010_06807_b200.ordering import partition_geometric
    from paper_2010_06807_b200.problems import make_config
    g = np.load(os.path.join(golden_dir, "ranks_C5_n48_L8.npz"))["ranks"]
    A, dims, L, eps, b, tol = make_config("C5", n=48)
    F = factorize(A, partition_geometric(dims, L), eps=eps)
    got = {(int(l), int(p)): (int(r), int(bf)) for l, p, bf, r in F.sparsify_log}
    bad = [(int(l), int(p), int(r), int(bf), got.get((int(l), int(p))))
           for l, p, r, bf in g if got.get((int(l), int(p))) != (int(r), int(bf))]
    assert not bad, f"{len(bad)} of {len(g)} interfaces differ, e.g. {bad[:5]}"


def test_speculative_flags_verified_and_equal_exact_mode():
    """Speculative row flags (no host read-back per factor wave) are checked
    on the device; with no mismatch the factorization equals the exact-flag
    mode: same ranks, row_of_col, stats and R_ss."""
    from paper_2010_06807_b200.factor import BlockHouseholder, factorize
    from paper_2010_06807_b200.ordering import partition_geometric
    from paper_2010_06807_b200.problems import make_config
    A, dims, L, eps, b, tol = make_config("C3", n=48)
    tree = partition_geometric(dims, L)
    Fs = factorize(A, tree, eps=eps)
    hs = Fs.device_timings()["host"]
    assert hs["speculate"] == 1 and hs["verified_blocks"] > 0 and hs["spec_mismatch"] == 0
    Fe = factorize(A, tree, eps=eps, _speculate=False)
    he = Fe.device_timings()["host"]
    assert he["speculate"] == 0 and he["verified_blocks"] == 0
    assert he["syncs"] > hs["syncs"]
    assert Fs.sparsify_log == Fe.sparsify_log
    assert np.array_equal(Fs.row_of_col, Fe.row_of_col)
    for a, c in zip(Fs.stats, Fe.stats):
        for key in ("n_factored", "factored_cols", "n_sparsified", "fine_retired", "cols_after",
                    "trailing_blocks"):
            assert a[key] == c[key], (a["level"], key)
        # exact zeros born of cancellation depend on rounding (batching)
        assert abs(a["trailing_nnz"] - c["trailing_nnz"]) <= 0.01 * c["trailing_nnz"]
    bs = [r for r in Fs.q_chain if isinstance(r, BlockHouseholder)]
    be = [r for r in Fe.q_chain if isinstance(r, BlockHouseholder)]
    assert len(bs) == len(be)
    for x, y in zip(bs, be):
        assert np.abs(x.R_ss - y.R_ss).max() <= 1e-10 * np.abs(y.R_ss).max()


def test_device_gmres_matches_host_loop():
    """spq_gmres (whole Arnoldi loop in HBM) against the host restatement of
    solve.py:66-209 (oracle/krylov.py) driving the same B200 chains:
    iterations within 1, final residual within 10x, solutions agreeing;
    restarted GMRES, an initial guess and a zero right-hand side too."""
    from oracle.krylov import gmres_host
    from paper_2010_06807_b200.factor import factorize
    from paper_2010_06807_b200.ordering import partition_geometric
    from paper_2010_06807_b200.problems import make_config
    from paper_2010_06807_b200.solve import gmres
    from paper_2010_06807_b200.sparse import matvec
    A, dims, L, eps, b, tol = make_config("C3", n=48)
    tree = partition_geometric(dims, L)
    F = factorize(A, tree, eps=eps)
    for kw in ({}, {"restart": 2}, {"x0": np.full(A.ncols, 0.5)}):
        xd, rd = gmres(A, b, F, tol=tol, **kw)
        xh, its, hist, conv = gmres_host(A, b, F, tol=tol, matvec=matvec, **kw)
        assert rd.meta.get("device")
        assert abs(rd.iterations - its) <= 1, kw
        assert len(rd.residuals) == rd.iterations + 1
        assert rd.converged == conv
        assert rd.final_residual <= 10 * max(hist[-1], 1e-16), kw
        np.testing.assert_allclose(rd.residuals[:2], hist[:2], rtol=1e-6)
        r = np.linalg.norm(b - matvec(A, xd)) / np.linalg.norm(b)
        assert r <= 10 * max(hist[-1], 1e-16)
        assert np.abs(xd - xh).max() <= 1e-8 * np.abs(xh).max()
    x0, r0 = gmres(A, np.zeros(A.ncols), F, tol=tol)
    assert r0.iterations == 0 and r0.converged and not x0.any()
    # maxit cap honoured, not converged
    x1, r1 = gmres(A, b, F, tol=1e-30, maxit=3)
    assert r1.iterations == 3 and not r1.converged and len(r1.residuals) == 4


def test_ill_conditioned_interface_raises():
    """Unscaled route: an interface whose column stack [A_pp; A_np] is
    numerically rank deficient (two identical columns) raises
    IllConditionedInterfaceError like the reference (factor.py:557-563);
    run in the build container, the reference raises it for interface 36
    (sigma_min 4.7e-18 below the floor 1.5e-14) on this input."""
    from paper_2010_06807_b200.errors import IllConditionedInterfaceError
    from paper_2010_06807_b200.factor import factorize
    from paper_2010_06807_b200.ordering import partition_geometric
    from paper_2010_06807_b200.problems import make_config
    from paper_2010_06807_b200.sparse import SparseMat
    A0, dims, L, eps, b, tol = make_config("C1")
    tree = partition_geometric(dims, L)
    c = sorted(tree.sparsify_at(4), key=lambda c: c.id)[0]
    D = A0.to_dense()
    D[:, int(c.cols[1])] = D[:, int(c.cols[0])]
    A = SparseMat.from_dense(D)
    with pytest.raises(IllConditionedInterfaceError) as ei:
        factorize(A, partition_geometric(dims, L), eps=eps, mode="unscaled")
    assert ei.value.interface == 36
    assert ei.value.sigma_min < 1e-14


@pytest.mark.parametrize("name,cfg,n,opts", [
    ("C3_n48_variant1", "C3", 48, {"mode": "variant1"}),
    ("C3_n48_variant2", "C3", 48, {"mode": "variant2"}),
    ("C1_variant1_se2", "C1", None, {"mode": "variant1", "scale_every": 2}),
    ("C1_variant2_se2", "C1", None, {"mode": "variant2", "scale_every": 2}),
])
def test_variant_targets_match_reference(name, cfg, n, opts):
    """The one-sided ('variant1': M = A_np^T) and Gram ('variant2') targets
    (factor.py:541-551): scaled apply on scaled levels, unscaled apply
    without rank enforcement on the others; against the live reference's
    goldens."""
    g = load(name)
    A, b, F, x, rep = _run(name, cfg, n, **opts)
    _check_against_reference(F, rep, g)


@pytest.mark.parametrize("cfg,n", [("C1", 24), ("C3", 48), ("C4", 12)])
def test_fill_within_symbolic_prediction(cfg, n, golden_dir):
    """The device path creates blocks only where the reference's symbolic
    elimination predicts fill (reference test tests/test_factor.py:168-183):
    at every level of the drop-free factorization, the live block keys are a
    subset of the golden `symbolic_fill_levels` pattern of the live reference."""
    import os
    from paper_2010_06807_b200.factor import factorize
    from paper_2010_06807_b200.ordering import partition_geometric
    from paper_2010_06807_b200.problems import make_config
    g = np.load(os.path.join(golden_dir, "symbolic.npz"))
    A, dims, L, eps, b, tol = make_config(cfg, n=n)
    tree = partition_geometric(dims, L)
    seen = {}

    class Obs:
        def on_level(self, state, lev, st):
            seen[lev] = state.trailing_keys()

    factorize(A, tree, eps=eps, sparsify=False, observer=Obs())
    assert sorted(seen) == list(range(1, L + 1))
    for lev, keys in seen.items():
        ref = {tuple(p) for p in g[f"{cfg}_n{n}_L{lev}"].tolist()}
        assert keys <= ref, (lev, sorted(keys - ref)[:5])
