"""TEST INFRASTRUCTURE ONLY — host restatement of the reference's GMRES.

Comparator for the device GMRES (``spq_gmres``): the same right-preconditioned
iteration as `pkg/src/nestqr/solve.py:66-209`, written as a small Arnoldi
object plus a Givens least-squares object.  Semantics it keeps (each tied to
the reference line range):

* operator v -> apply_qt(A solve_w(v)); starting residual z = apply_qt(b - A x)
  (`solve.py:98-131`);
* modified Gram-Schmidt, then ONE extra re-orthogonalisation pass when
  max|Q^T w| / ||w|| > 1e-8 (`solve.py:145-165`);
* Givens rotations of the Hessenberg column, least-squares residual |g_{j+1}|
  (`solve.py:166-180`);
* every iteration forms x_j = x + solve_w(Q y) and records the TRUE relative
  residual; converge on |g_{j+1}|/||b|| <= tol or true residual <= tol; the
  best iterate is returned (`solve.py:181-209`);
* restarts after ``restart`` inner steps, ``maxit`` caps the total.

Only ``tests/`` import this (see ``oracle/__init__.py``).
"""

from __future__ import annotations

import numpy as np
from scipy.linalg import solve_triangular

REORTH = 1e-8


class _Arnoldi:
    """Orthonormal Krylov basis with MGS + conditional re-orthogonalisation."""

    def __init__(self, n, m, z):
        self.Q = np.zeros((n, m + 1))
        self.beta = float(np.linalg.norm(z))
        self.Q[:, 0] = z / self.beta

    def extend(self, j, w):
        """Orthogonalise w against Q[:, :j+1]; returns (h[0..j+1], w_next)."""
        Qj = self.Q[:, :j + 1]
        h = np.zeros(j + 2)
        for i in range(j + 1):
            h[i] = Qj[:, i] @ w
            w = w - h[i] * Qj[:, i]
        nw = float(np.linalg.norm(w))
        if nw > 0.0:
            extra = Qj.T @ w
            if np.max(np.abs(extra)) / nw > REORTH:
                h[:j + 1] += extra
                w = w - Qj @ extra
                nw = float(np.linalg.norm(w))
        h[j + 1] = nw
        return h, w


class _GivensLS:
    """Upper-triangular least-squares min ||beta e1 - H y|| by Givens rotations."""

    def __init__(self, m, beta):
        self.R = np.zeros((m + 1, m))
        self.c = np.zeros(m)
        self.s = np.zeros(m)
        self.g = np.zeros(m + 1)
        self.g[0] = beta

    def push(self, j, h):
        col = h.copy()
        for i in range(j):
            a, b = col[i], col[i + 1]
            col[i] = self.c[i] * a + self.s[i] * b
            col[i + 1] = -self.s[i] * a + self.c[i] * b
        r = float(np.hypot(col[j], col[j + 1]))
        if r == 0.0:
            self.c[j], self.s[j] = 1.0, 0.0
        else:
            self.c[j], self.s[j] = col[j] / r, col[j + 1] / r
        col[j] = self.c[j] * col[j] + self.s[j] * col[j + 1]
        col[j + 1] = 0.0
        self.R[:j + 2, j] = col
        self.g[j + 1] = -self.s[j] * self.g[j]
        self.g[j] = self.c[j] * self.g[j]
        return abs(self.g[j + 1])

    def solve(self, j):
        return solve_triangular(self.R[:j + 1, :j + 1], self.g[:j + 1], lower=False)


def gmres_host(A, b, F, tol=1e-12, maxit=300, restart=None, x0=None, matvec=None):
    """Returns (x_best, iterations, history, converged)."""
    if matvec is None:
        def matvec(M, v):
            return M @ v
    b = np.asarray(b, dtype=np.float64)
    n = b.shape[0]
    bn = float(np.linalg.norm(b))
    if bn == 0.0:
        return np.zeros(n), 0, np.array([0.0]), True
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64)

    def true_res(v):
        return float(np.linalg.norm(b - matvec(A, v))) / bn

    hist = [true_res(x)]
    best = (hist[0], x)
    conv = hist[0] <= tol
    its = 0
    while not conv and its < maxit:
        z = F.apply_qt(b - matvec(A, x))
        if float(np.linalg.norm(z)) == 0.0:
            conv = True
            break
        m = maxit - its if restart is None else min(restart, maxit - its)
        kr = _Arnoldi(n, m, z)
        ls = _GivensLS(m, kr.beta)
        x_cycle = x
        for j in range(m):
            h, w = kr.extend(j, F.apply_qt(matvec(A, F.solve_w(kr.Q[:, j]))))
            est = ls.push(j, h)
            x_cycle = x + F.solve_w(kr.Q[:, :j + 1] @ ls.solve(j))
            its += 1
            hist.append(true_res(x_cycle))
            if hist[-1] < best[0]:
                best = (hist[-1], x_cycle)
            if est / bn <= tol or hist[-1] <= tol:
                conv = True
                break
            if h[j + 1] <= 1e-300:
                break
            kr.Q[:, j + 1] = w / h[j + 1]
        x = x_cycle
    return best[1], its, np.asarray(hist), bool(conv)
