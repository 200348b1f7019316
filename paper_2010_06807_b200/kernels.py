"""The reference's dense-kernel plugin API, served by the sm_100a library.

Mirrors `pkg/src/nestqr/kernels/__init__.py:73-241` — same names, argument
meaning, return types and error behaviour — so the reference's kernel tests
(`pkg/tests/test_kernels.py`) read unchanged against this module.  Every
call runs on the device through the C-ABI (one problem per call: this is the
per-kernel parity surface; the factorization itself batches).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._lib import Context
from .errors import NestqrError, SingularPivotError

PIVOT_FLOOR = 1e-14
_ctx = None


def _context():
    global _ctx
    if _ctx is None:
        _ctx = Context()
    return _ctx


def backend_name():
    return "b200"


def set_backend(name):
    if name.strip().lower() != "b200":
        raise NestqrError(f"unknown kernel backend {name!r} (this package only has 'b200')")
    return "b200"


@dataclass
class HouseholderPanel:
    V: np.ndarray
    tau: np.ndarray
    T: np.ndarray
    rows: np.ndarray | None = None

    @property
    def m(self):
        return self.V.shape[0]

    @property
    def k(self):
        return self.V.shape[1]

    @property
    def payload_scalars(self):
        return self.V.size + self.tau.size + self.T.size

    def apply(self, C, transpose=False, overwrite=False):
        C = np.asarray(C, dtype=np.float64)
        if C.shape[0] != self.m:
            raise NestqrError(f"panel expects leading dim {self.m}, got {C.shape[0]}")
        if self.k == 0:
            return C if overwrite else C.copy()
        vec = C.ndim == 1
        B = np.ascontiguousarray(C.reshape(self.m, -1), dtype=np.float64).copy()
        _context().call("spq_apply_panel", self.m, self.k, B.shape[1],
                        np.ascontiguousarray(self.V), np.ascontiguousarray(self.T), B,
                        int(bool(transpose)))
        if overwrite and not vec and C.flags.c_contiguous:
            C[...] = B
            return C
        return B[:, 0] if vec else B


@dataclass
class RRQRResult:
    panel: HouseholderPanel
    R: np.ndarray
    resid: np.ndarray
    perm: np.ndarray
    rank: int

    def q_dense(self):
        return self.panel.apply(np.eye(self.panel.m))

    @property
    def Q(self):
        return self.q_dense()


def qr_house(B):
    """Householder QR of a tall block (reference `kernels/__init__.py:147-166`)."""
    B = np.ascontiguousarray(B, dtype=np.float64)
    m, k = B.shape
    if m < k:
        raise NestqrError(f"qr_house needs m >= k, got {B.shape}")
    V = np.zeros((m, k))
    tau = np.zeros(k)
    T = np.zeros((k, k))
    R = np.zeros((k, k))
    if k:
        _context().call("spq_qr_house", m, k, B, V, tau, T, R)
    return HouseholderPanel(V=V, tau=tau, T=T), R


def apply_panel_left(panel, C, transpose=False, overwrite=False):
    return panel.apply(C, transpose=transpose, overwrite=overwrite)


def rrqr_threshold(M, eps, min_rank=0):
    """Threshold column-pivoted QR (reference `kernels/__init__.py:174-199`)."""
    if not (0.0 <= eps < 1.0):
        raise NestqrError(f"rrqr_threshold needs eps in [0, 1), got {eps}")
    M = np.ascontiguousarray(M, dtype=np.float64)
    m, k = M.shape
    min_rank = min(int(min_rank), min(m, k))
    kmax = min(m, k)
    V = np.zeros((m, max(kmax, 0)))
    tau = np.zeros(max(kmax, 0))
    Tred = M.copy()
    perm = np.arange(k, dtype=np.int64)
    import ctypes as C
    r = C.c_int64(0)
    if m and k:
        _context().call("spq_rrqr", m, k, M, float(eps), int(min_rank), V, tau, Tred, perm,
                        C.byref(r))
    r = int(r.value)
    V = np.ascontiguousarray(V[:, :r])
    tau = tau[:r].copy()
    T = _build_t(V, tau)
    return RRQRResult(panel=HouseholderPanel(V=V, tau=tau, T=T), R=np.array(Tred[:r, :]),
                      resid=np.array(Tred[r:, r:]), perm=perm, rank=r)


def build_t(V, tau):
    """Compact-WY T of (V, tau) on the device (the backend contract's
    ``build_t``, reference `kernels/_numba.py:101-117`)."""
    V = np.ascontiguousarray(V, dtype=np.float64)
    k = V.shape[1]
    T = np.zeros((k, k))
    if k:
        _context().call("spq_build_t", V.shape[0], k, V, np.ascontiguousarray(tau, np.float64), T)
    return T


_build_t = build_t


def tri_solve(R, C, side="left"):
    """R^{-1} C (left) or C R^{-1} (right) (reference `kernels/__init__.py:202-233`)."""
    R = np.ascontiguousarray(R, dtype=np.float64)
    C = np.ascontiguousarray(C, dtype=np.float64)
    k = R.shape[0]
    if k == 0:
        return C.copy()
    if side not in ("left", "right"):
        raise NestqrError(f"tri_solve side must be 'left' or 'right', got {side!r}")
    vec = C.ndim == 1
    if side == "left":
        B = C.reshape(k, -1)
        X = np.empty_like(B)
        _context().call("spq_tri_solve", k, B.shape[1], R, np.ascontiguousarray(B), 0, X)
        return X[:, 0] if vec else X
    B = C.reshape(-1, k) if not vec else C.reshape(1, k)
    X = np.empty_like(B)
    _context().call("spq_tri_solve", k, B.shape[0], R, np.ascontiguousarray(B), 1, X)
    return X[0] if vec else X


def spectral_norm(A):
    """sigma_max (reference `kernels/__init__.py:236-241`; stats only)."""
    A = np.asarray(A, dtype=np.float64)
    if A.size == 0:
        return 0.0
    return float(np.linalg.svd(A, compute_uv=False)[0])
