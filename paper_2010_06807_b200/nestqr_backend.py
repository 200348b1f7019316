"""Drop-in kernel backend for the reference package (`nestqr.kernels._impl`).

The reference selects its dense-kernel backend through a module global,
``nestqr.kernels._impl`` (`pkg/src/nestqr/kernels/__init__.py:26-67`); its own
tests swap that global (`pkg/tests/test_kernels.py:22-27`).  This module
implements that backend contract on the B200 -- the same five functions with
the same argument meaning and return layout as `kernels/_numba.py` /
`kernels/_numpy.py` -- so a maintainer injects it with

    import nestqr.kernels as K
    from paper_2010_06807_b200 import nestqr_backend
    K._impl = nestqr_backend

and every ``qr_house`` / ``rrqr_threshold`` / ``tri_solve`` call of the
reference then runs on the device.  Like the reference
backends, these functions do not validate: the wrappers in
``nestqr.kernels`` do (shape checks, the pivot floor).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import kernels as _k


def house_qr(B):
    """(V[m,k], tau[k], R[k,k]) of B (m >= k); `_numba.py:52-84`."""
    panel, R = _k.qr_house(B)
    return panel.V, panel.tau, R


def build_t(V, tau):
    """Upper-triangular compact-WY T; `_numba.py:101-117`."""
    return _k.build_t(V, tau)


def cpqr_threshold(M, eps, min_rank):
    """(V[m,r], tau[r], Tred[m,k], perm int64[k], r); `_numba.py:120-167`."""
    M = np.ascontiguousarray(M, dtype=np.float64)
    m, k = M.shape
    kmax = min(m, k)
    V = np.zeros((m, kmax))
    tau = np.zeros(kmax)
    Tred = M.copy()
    perm = np.arange(k, dtype=np.int64)
    r = C.c_int64(0)
    if m and k:
        _k._context().call("spq_rrqr", m, k, M, float(eps), int(min(min_rank, kmax)), V, tau,
                           Tred, perm, C.byref(r))
    r = int(r.value)
    return np.ascontiguousarray(V[:, :r]), tau[:r].copy(), Tred, perm, r


def tri_solve_left(R, C_):
    """R^{-1} C (R k x k upper, C k x n); `_numba.py:170-178`."""
    return _k.tri_solve(R, np.asarray(C_, dtype=np.float64).reshape(R.shape[0], -1), side="left")


def tri_solve_right(R, C_):
    """C R^{-1} (C n x k); `_numba.py:181-191`."""
    return _k.tri_solve(R, np.asarray(C_, dtype=np.float64).reshape(-1, R.shape[0]), side="right")
