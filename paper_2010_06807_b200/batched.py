"""BASELINE config 2: the isolated batched kernels (device-resident batches).

* ``batched_qr(Bs, Cs)`` — Householder QR of every block B_i (m_i x k_i,
  k_i <= m_i) and Q_i^T applied to its companion C_i, all blocks in one
  batch (`spq_batched_qr`; the same cluster panel kernel + DMMA compact-WY
  engine the factorization uses).  Semantics of the reference's
  ``qr_house`` + ``apply_panel_left(transpose=True)`` (`kernels/__init__.py:147-171`).
* ``batched_rrqr(Ms, eps)`` — threshold CPQR of every m x n block with the
  relative rule of ``rrqr_threshold`` (`kernels/__init__.py:174-199`), one
  CTA per block with the block resident in shared memory (`spq_batched_rrqr`).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import Context

_ctx = None


def _context():
    global _ctx
    if _ctx is None:
        _ctx = Context()
    return _ctx


def batched_qr(Bs, Cs):
    """Returns (list of R_i, list of H_i^T C_i, device ms)."""
    m = np.array([b.shape[0] for b in Bs], np.int64)
    k = np.array([b.shape[1] for b in Bs], np.int64)
    nc = np.array([c.shape[1] for c in Cs], np.int64)
    B = np.concatenate([np.asarray(b, np.float64).ravel(order="F") for b in Bs])
    Cp = np.concatenate([np.asarray(c, np.float64).ravel(order="F") for c in Cs])
    R = np.zeros(int((k * k).sum()))
    ms = C.c_float()
    _context().call("spq_batched_qr", len(Bs), m, k, nc, B, R, Cp, C.byref(ms))
    Rs, Co = [], []
    orr = oc = 0
    for i in range(len(Bs)):
        kk, mm, cc = int(k[i]), int(m[i]), int(nc[i])
        Rs.append(R[orr:orr + kk * kk].reshape((kk, kk), order="F"))
        Co.append(Cp[oc:oc + mm * cc].reshape((mm, cc), order="F"))
        orr += kk * kk
        oc += mm * cc
    return Rs, Co, float(ms.value)


def batched_rrqr(Ms, eps):
    """Returns (ranks, |R_ii| of accepted steps (nb x min(m,n)), device ms)."""
    Ms = np.asarray(Ms, np.float64)
    nb, m, n = Ms.shape
    Mp = np.ascontiguousarray(Ms.transpose(0, 2, 1)).ravel()   # column-major per block
    ranks = np.zeros(nb, np.int64)
    rdiag = np.zeros(nb * min(m, n))
    ms = C.c_float()
    _context().call("spq_batched_rrqr", nb, m, n, Mp, float(eps), ranks, rdiag, C.byref(ms))
    return ranks, rdiag.reshape(nb, min(m, n)), float(ms.value)


def config2_inputs(n_qr=4096, n_rrqr=4096, qr_seed=2, rrqr_seed=3):
    """Seeded synthetic inputs of BASELINE config 2: QR blocks with
    m ~ U{32..256}, k ~ U{16..128} clipped to k <= m, N(0,1) entries and an
    m x k companion; RRQR blocks U diag(10^(-j/8)) V^T (64 x 192)."""
    rng = np.random.default_rng(qr_seed)
    Bs, Cs = [], []
    for _ in range(n_qr):
        m = int(rng.integers(32, 257))
        k = min(int(rng.integers(16, 129)), m)
        Bs.append(rng.standard_normal((m, k)))
        Cs.append(rng.standard_normal((m, k)))
    rng = np.random.default_rng(rrqr_seed)
    sig = 10.0 ** (-np.arange(64) / 8.0)
    Ms = np.empty((n_rrqr, 64, 192))
    for i in range(n_rrqr):
        U, _ = np.linalg.qr(rng.standard_normal((64, 64)))
        W, _ = np.linalg.qr(rng.standard_normal((192, 64)))
        Ms[i] = (U * sig) @ W.T
    return Bs, Cs, Ms
