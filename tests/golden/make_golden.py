"""Generate the golden vectors from the REAL reference package.

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src:/root/repo NUMBA_CACHE_DIR=/tmp/nbc \
        python tests/golden/make_golden.py [--big]

Outputs (committed, small):
  kernels.npz   known-answer cases for qr_house / rrqr_threshold / tri_solve
                (reference `kernels/__init__.py:147-233`, numba backend)
  factor_<case>.npz  per-case factorization results: per-level stats, the
                per-interface rank sequence, row_of_col; diag(R_ss), max|R_sn|
                and ||R_sn||_F of every elimination record, full R_ss / R_sn of
                picked records; diag(R_pp) of every interface scaling, full R_pp
                of picks; rank and tau of every sparsifier, V/T of picks (and
                R_ff / R_fc / H_f tau in the unscaled branch); the reference's
                own apply_qt / solve_w / apply_w of a seeded vector; GMRES
                history; plus the numpy-backend divergence envelope of every
                one of those quantities, per record
  trees.json    tree digests of the reference's partition_geometric per config
--big adds the full C3 (256^2) and C4 (32^3) runs (minutes of CPU).
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import nestqr.kernels as K                                    # noqa: E402
from nestqr.factor import (BlockHouseholder, InterfaceScaling,  # noqa: E402
                           Sparsifier, factorize)
from nestqr.ordering import partition_geometric as ref_partition  # noqa: E402
from nestqr.solve import gmres                                 # noqa: E402
from nestqr.sparse import SparseMat                            # noqa: E402

from paper_2010_06807_b200.ordering import tree_digest         # noqa: E402
from paper_2010_06807_b200.problems import make_config         # noqa: E402

CASES = {
    # name: (config, n override, factorize options)
    "C1_n24": ("C1", 24, {}),
    "C1": ("C1", None, {}),
    "C3_n48": ("C3", 48, {}),
    "C4_n12": ("C4", 12, {}),
    # the unscaled sparsification branch and alternating scaling
    # (factor.py:557-566, 660-709, 849-850)
    "C1_unscaled": ("C1", None, {"mode": "unscaled"}),
    "C3_n48_unscaled": ("C3", 48, {"mode": "unscaled"}),
    "C1_se2": ("C1", None, {"scale_every": 2}),
    "C3_n48_se2": ("C3", 48, {"scale_every": 2}),
    "C4_n12_unscaled": ("C4", 12, {"mode": "unscaled"}),
    "C3_n96_unscaled": ("C3", 96, {"mode": "unscaled"}),
    "C3_n96_se2": ("C3", 96, {"scale_every": 2}),
    # one-sided / Gram compression targets (factor.py:541-551)
    "C3_n48_variant1": ("C3", 48, {"mode": "variant1"}),
    "C3_n48_variant2": ("C3", 48, {"mode": "variant2"}),
    "C1_variant1_se2": ("C1", None, {"mode": "variant1", "scale_every": 2}),
    "C1_variant2_se2": ("C1", None, {"mode": "variant2", "scale_every": 2}),
}
# full-size metric configs; the numpy-backend envelope run is part of them
BIG = {"C3": ("C3", None, {}), "C4": ("C4", None, {})}


def kernel_cases():
    rng = np.random.default_rng(2024)
    out = {}
    shapes = [(1, 1), (2, 1), (7, 7), (20, 5), (64, 40), (130, 33), (200, 96), (37, 36)]
    for t, (m, k) in enumerate(shapes):
        B = rng.standard_normal((m, k))
        if t == 3:
            B[:, 2] = 0.0                       # zero column -> tau = 0
        if t == 4:
            B[5:, 7] = 0.0
            B[:5, 7] = -1.0                     # sigma != 0, alpha < 0
        if t == 5:
            B[1:, 0] = 0.0
            B[0, 0] = -3.0                      # sigma == 0, alpha < 0 -> tau = 2
        panel, R = K.qr_house(B)
        C = rng.standard_normal((m, 3))
        out[f"qr{t}_B"] = B
        out[f"qr{t}_V"] = panel.V
        out[f"qr{t}_tau"] = panel.tau
        out[f"qr{t}_T"] = panel.T
        out[f"qr{t}_R"] = R
        out[f"qr{t}_C"] = C
        out[f"qr{t}_HtC"] = K.apply_panel_left(panel, C, transpose=True)
    rr = []
    for t in range(8):
        m, k = [(12, 9), (30, 80), (64, 192), (10, 14), (50, 50), (8, 8), (40, 300), (5, 3)][t]
        if t in (2, 6):
            U, _ = np.linalg.qr(rng.standard_normal((m, m)))
            W, _ = np.linalg.qr(rng.standard_normal((k, m)))
            M = U @ np.diag(10.0 ** (-np.arange(m) / 8.0)) @ W.T
        elif t == 5:
            M = np.outer(rng.standard_normal(m), rng.standard_normal(k))
        else:
            M = rng.standard_normal((m, k)) @ np.diag(10.0 ** -np.linspace(0, 9, k))
        for e, eps in enumerate([0.0, 1e-8, 1e-4, 1e-2, 0.5]):
            res = K.rrqr_threshold(M, eps)
            key = f"rr{t}_{e}"
            out[f"rr{t}_M"] = M
            out[key + "_eps"] = np.float64(eps)
            out[key + "_rank"] = np.int64(res.rank)
            out[key + "_perm"] = res.perm
            out[key + "_R"] = res.R
            out[key + "_V"] = res.panel.V
            out[key + "_tau"] = res.panel.tau
            rr.append(key)
    for t, k in enumerate([1, 5, 33, 70]):
        Rm = np.triu(rng.standard_normal((k, k))) + 4 * np.eye(k)
        C = rng.standard_normal((k, 4))
        Cr = rng.standard_normal((9, k))
        out[f"ts{t}_R"] = Rm
        out[f"ts{t}_C"] = C
        out[f"ts{t}_Cr"] = Cr
        out[f"ts{t}_left"] = K.tri_solve(Rm, C, side="left")
        out[f"ts{t}_right"] = K.tri_solve(Rm, Cr, side="right")
    out["n_qr"] = np.int64(len(shapes))
    out["rr_keys"] = np.array(rr)
    out["n_ts"] = np.int64(4)
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **out)


class RankLog:
    """observer: record (level, interface id, cols before, cols after)."""

    def __init__(self):
        self.rows = []
        self.lev = None

    def on_sparsify(self, state, p, when):
        if when == "before":
            self._b = len(state.cols_of[p])
        else:
            self.rows.append((p, self._b, len(state.cols_of[p])))


PICK_MAX = 160_000          # largest full block stored for a picked record


def _rel(a, c):
    """max|a - c| / max|c| (inf on a shape mismatch)."""
    if a.shape != c.shape:
        return np.inf
    if a.size == 0:
        return 0.0
    return float(np.abs(a - c).max() / max(np.abs(c).max(), 1e-300))


def _picks(n):
    return sorted(set(i for i in (0, 1, n // 2, n - 2, n - 1) if 0 <= i < n))


def _records(F):
    bh = [r for r in F.q_chain if isinstance(r, BlockHouseholder)]
    isc = [r for r in F.q_chain if isinstance(r, InterfaceScaling)]
    sp = [r for r in F.q_chain if isinstance(r, Sparsifier)]
    return bh, isc, sp


def _chain_vectors(F, N):
    v = np.random.default_rng(11).standard_normal(N)
    return {"apply_qt": F.apply_qt(v), "solve_w": F.solve_w(v), "apply_w": F.apply_w(v)}


class KeyLog:
    """Cluster id of every record, per kind, in chain order (wraps the
    reference's TrailingState level operations; results untouched)."""

    def __init__(self):
        import nestqr.factor as NF
        self.keys = {"bh": [], "is": [], "sp": []}
        TS = NF.TrailingState
        self._orig = (TS.factor_interior, TS.scale_interface, TS.sparsify_interface)
        log = self.keys
        fi, si, spi = self._orig

        def factor_interior(st, s):
            rec = fi(st, s)
            if rec is not None:
                log["bh"].append(s)
            return rec

        def scale_interface(st, p):
            rec = si(st, p)
            if rec is not None:
                log["is"].append(p)
            return rec

        def sparsify_interface(st, p, *a, **k):
            rec, dropped = spi(st, p, *a, **k)
            if rec is not None:
                log["sp"].append(p)
            return rec, dropped

        TS.factor_interior, TS.scale_interface = factor_interior, scale_interface
        TS.sparsify_interface = sparsify_interface
        self._TS = TS

    def close(self):
        self._TS.factor_interior, self._TS.scale_interface, self._TS.sparsify_interface = self._orig


def factor_case(name, cfg, n, envelope=None, **opts):
    A0, dims, L, eps, b, tol = make_config(cfg, n=n)
    A = SparseMat(A0.nrows, A0.ncols, A0.indptr, A0.indices, A0.data)
    tree = ref_partition(dims, L)
    K.set_backend("numba")
    log = RankLog()
    klog = KeyLog()
    t0 = time.perf_counter()
    try:
        F = factorize(A, tree, eps=eps, observer=log, **opts)
    finally:
        klog.close()
    t_fac = time.perf_counter() - t0
    t0 = time.perf_counter()
    x, rep = gmres(A, b, F, tol=tol)
    t_sol = time.perf_counter() - t0
    out = {"dims": np.array(dims), "L": np.int64(L), "eps": np.float64(eps),
           "tol": np.float64(tol), "t_factor": np.float64(t_fac),
           "t_gmres": np.float64(t_sol)}
    out["options"] = np.array(json.dumps(opts))
    keys = [k for k in F.stats[0] if not k.startswith("t_")]
    out["stat_keys"] = np.array(keys)
    out["stats"] = np.array([[float(s[k]) for k in keys] for s in F.stats])
    out["sparsify_log"] = np.array(log.rows, dtype=np.int64).reshape(-1, 3)
    out["row_of_col"] = F.row_of_col
    out["payload"] = np.int64(F.payload_scalars)
    bh, isc, sp = _records(F)
    # cluster id of every record (records of independent clusters commute, so
    # the device's chain order may differ; the comparison matches by id)
    out["bh_key"] = np.array(klog.keys["bh"], dtype=np.int64)
    out["rpp_key"] = np.array(klog.keys["is"], dtype=np.int64)
    out["sp_key"] = np.array(klog.keys["sp"], dtype=np.int64)
    assert len(out["bh_key"]) == len(bh) and len(out["rpp_key"]) == len(isc)
    assert len(out["sp_key"]) == len(sp)
    # ---- elimination records (factor.py:486-493): R_ss, R_sn
    out["rss_diag"] = np.concatenate([np.diag(r.R_ss) for r in bh])
    out["rss_k"] = np.array([r.R_ss.shape[0] for r in bh])
    out["rsn_shape"] = np.array([r.R_sn.shape for r in bh], dtype=np.int64).reshape(-1, 2)
    out["rsn_maxabs"] = np.array([np.abs(r.R_sn).max(initial=0.0) for r in bh])
    out["rsn_fro"] = np.array([np.linalg.norm(r.R_sn) for r in bh])
    pick = sorted(i for i in _picks(len(bh)) if bh[i].R_ss.shape[0] <= 256)
    out["rss_pick"] = np.array(pick)
    for i in pick:
        out[f"rss_{i}"] = bh[i].R_ss
        out[f"rsn_{i}_shape"] = np.array(bh[i].R_sn.shape)
        out[f"rsn_{i}_fro"] = np.float64(np.linalg.norm(bh[i].R_sn))
    rsn_pick = [i for i in pick if bh[i].R_sn.size <= PICK_MAX]
    out["rsn_pick"] = np.array(rsn_pick, dtype=np.int64)
    for i in rsn_pick:
        out[f"rsn_{i}"] = bh[i].R_sn
    # ---- interface scaling records (factor.py:504-532): R_pp
    out["rpp_k"] = np.array([r.R_pp.shape[0] for r in isc], dtype=np.int64)
    out["rpp_diag"] = (np.concatenate([np.diag(r.R_pp) for r in isc]) if isc
                       else np.zeros(0))
    out["rpp_fro"] = np.array([np.linalg.norm(r.R_pp) for r in isc])
    pp_pick = [i for i in _picks(len(isc)) if isc[i].R_pp.size <= PICK_MAX]
    out["rpp_pick"] = np.array(pp_pick, dtype=np.int64)
    for i in pp_pick:
        out[f"rpp_{i}"] = isc[i].R_pp
    # ---- sparsifier records (factor.py:627-709): rank, tau, V; R_ff/R_fc unscaled
    out["sp_rank"] = np.array([r.rank for r in sp], dtype=np.int64)
    out["sp_scaled"] = np.array([bool(r.scaled) for r in sp])
    out["sp_m"] = np.array([len(r.cols) for r in sp], dtype=np.int64)
    out["sp_tau"] = (np.concatenate([r.q_panel.tau for r in sp]) if sp else np.zeros(0))
    out["sp_ntau"] = np.array([len(r.q_panel.tau) for r in sp], dtype=np.int64)
    sp_pick = [i for i in _picks(len(sp)) if sp[i].q_panel.V.size <= PICK_MAX]
    out["sp_pick"] = np.array(sp_pick, dtype=np.int64)
    for i in sp_pick:
        out[f"sp_{i}_V"] = sp[i].q_panel.V
        out[f"sp_{i}_T"] = sp[i].q_panel.T
    unsc = [i for i, r in enumerate(sp) if not r.scaled]
    if unsc:
        out["rff_k"] = np.array([sp[i].R_ff.shape[0] for i in unsc], dtype=np.int64)
        out["rff_diag"] = np.concatenate([np.diag(sp[i].R_ff) for i in unsc])
        out["rfc_fro"] = np.array([np.linalg.norm(sp[i].R_fc) for i in unsc])
        out["hf_tau"] = np.concatenate([sp[i].hf_panel.tau for i in unsc])
        out["unsc_idx"] = np.array(unsc, dtype=np.int64)
        for i in _picks(len(unsc)):
            j = unsc[i]
            if sp[j].R_ff.size + sp[j].R_fc.size <= PICK_MAX:
                out[f"rff_{j}"] = sp[j].R_ff
                out[f"rfc_{j}"] = sp[j].R_fc
    out["chain_kinds"] = np.array([type(r).__name__ for r in F.q_chain[:-1]])
    # ---- the reference's own chain applications (factor.py:281-300)
    for k, v in _chain_vectors(F, A.ncols).items():
        out[f"chain_{k}"] = v
    out["gmres_iters"] = np.int64(rep.iterations)
    out["gmres_hist"] = rep.residuals
    out["gmres_converged"] = np.bool_(rep.converged)
    out["x_norm"] = np.float64(np.linalg.norm(x))
    # rounding envelope (F3): numpy backend on the same inputs
    if envelope is None:
        envelope = A.ncols <= 16384
    if envelope:
        K.set_backend("numpy")
        t0 = time.perf_counter()
        F2 = factorize(A, tree, eps=eps, **opts)
        out["t_factor_numpy"] = np.float64(time.perf_counter() - t0)
        # structure decided by exact zeros (panel rows with any nonzero,
        # trailing_nnz) is itself rounding-dependent: the numpy twin's values
        out["payload_numpy"] = np.int64(F2.payload_scalars)
        out["stats_numpy"] = np.array([[float(s_[k]) for k in keys] for s_ in F2.stats])
        K.set_backend("numba")
        bh2, isc2, sp2 = _records(F2)
        out["rss_envelope"] = np.array([_rel(a.R_ss, c.R_ss) for a, c in zip(bh2, bh)])
        out["rsn_envelope"] = np.array([_rel(a.R_sn, c.R_sn) for a, c in zip(bh2, bh)])
        out["rpp_envelope"] = np.array([_rel(a.R_pp, c.R_pp) for a, c in zip(isc2, isc)])
        out["sp_envelope"] = np.array([_rel(a.q_panel.V, c.q_panel.V) for a, c in zip(sp2, sp)])
        out["sp_rank_numpy"] = np.array([r.rank for r in sp2], dtype=np.int64)
        if unsc:
            out["rff_envelope"] = np.array([_rel(sp2[i].R_ff, sp[i].R_ff) if i < len(sp2)
                                            and not sp2[i].scaled else np.inf for i in unsc])
        ch2 = _chain_vectors(F2, A.ncols)
        for k, v in ch2.items():
            out[f"chain_{k}_envelope"] = np.float64(_rel(v, out[f"chain_{k}"]))
    np.savez_compressed(os.path.join(HERE, f"factor_{name}.npz"), **out)
    print(f"{name}: N={A.ncols} L={L} factor {t_fac:.2f}s gmres {t_sol:.2f}s "
          f"its={rep.iterations} res={rep.final_residual:.3e} "
          f"records bh={len(bh)} is={len(isc)} sp={len(sp)} (unscaled {len(unsc)})", flush=True)


def trees():
    dig = {}
    for cfg, dims, L in [("C1", (64, 64), 6), ("C3", (256, 256), 10),
                         ("C4", (32, 32, 32), 9), ("C5", (64, 64, 64), 11),
                         ("C1_n24", (24, 24), 4), ("C3_n48", (48, 48), 6),
                         ("C4_n12", (12, 12, 12), 5), ("odd", (20, 37), 4),
                         ("odd3", (12, 9, 17), 4)]:
        dig[cfg] = {"dims": list(dims), "L": L, "sha256": tree_digest(ref_partition(dims, L))}
    with open(os.path.join(HERE, "trees.json"), "w") as fh:
        json.dump(dig, fh, indent=1)


if __name__ == "__main__":
    trees()
    kernel_cases()
    cases = dict(CASES)
    if "--big" in sys.argv:
        cases.update(BIG)
    only = [a for a in sys.argv[1:] if not a.startswith("--")]
    for name, (cfg, n, opts) in cases.items():
        if only and name not in only:
            continue
        factor_case(name, cfg, n, envelope=True if name in BIG else None, **opts)
