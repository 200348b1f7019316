"""Seeded upwind convection-diffusion generators for the benchmark configs.

BASELINE.json configs 1/3/4/5 ask for first-order UPWIND finite differences
with a vector advection field and per-cell coefficients; the reference's
generator (`pkg/src/nestqr/problems.py:118-184`) is centred with an
isotropic scalar field, so it cannot produce them.  This module
is the documented replacement; the factorization consumes its output exactly
like any other square CSC matrix.

Discretisation of  -div(kappa grad u) + beta . grad u  on the n^d interior
nodes of the unit cube, h = 1/(n+1), homogeneous Dirichlet boundary:

* diffusion: the face between nodes a and b carries the harmonic mean
  2 k_a k_b / (k_a + k_b); a boundary face carries the node's own kappa
  (as the reference does, `problems.py:154-165`);
* convection, per axis and per node with beta_x taken AT the node:
  beta_x > 0 -> beta_x (u_i - u_{i-1}) / h,  beta_x < 0 -> beta_x (u_{i+1} - u_i) / h.
  Couplings to boundary nodes vanish (u = 0 there).

Unknowns follow C-order raveling of the (x, y[, z]) grid, matching the
geometric partitioner (`ordering.partition_geometric`).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import NestqrError
from .sparse import SparseMat


@dataclass(frozen=True)
class UpwindSpec:
    n: int
    ndim: int = 2
    kappa: str = "const"          # "const" | "loguniform"
    kappa_const: float = 1.0
    kappa_range: tuple = (0.1, 10.0)
    beta: str = "const"           # "const" | "uniform"
    beta_const: tuple = (20.0, 20.0)
    beta_range: float = 50.0      # per-component U(-beta_range, beta_range)
    seed: int = 0

    @property
    def dims(self):
        return (self.n,) * self.ndim

    @property
    def N(self):
        return self.n ** self.ndim


def _fields(spec):
    d = spec.ndim
    rng = np.random.default_rng(spec.seed)
    if spec.kappa == "const":
        kappa = np.full(spec.dims, float(spec.kappa_const))
    elif spec.kappa == "loguniform":
        lo, hi = (math.log10(v) for v in spec.kappa_range)
        kappa = 10.0 ** rng.uniform(lo, hi, size=spec.dims)
    else:
        raise NestqrError(f"unknown kappa field {spec.kappa!r}")
    if spec.beta == "const":
        bc = np.asarray(spec.beta_const, dtype=np.float64)
        if bc.shape != (d,):
            raise NestqrError(f"beta_const needs {d} components")
        beta = np.broadcast_to(bc, spec.dims + (d,)).copy()
    elif spec.beta == "uniform":
        beta = rng.uniform(-spec.beta_range, spec.beta_range, size=spec.dims + (d,))
    else:
        raise NestqrError(f"unknown beta field {spec.beta!r}")
    return kappa, beta


def upwind_convection_diffusion(spec):
    """Assemble the upwind system matrix (SparseMat, N x N, 5/7-point)."""
    n, d = spec.n, spec.ndim
    if n < 2 or d not in (2, 3):
        raise NestqrError(f"bad grid n={n}, ndim={d}")
    h = 1.0 / (n + 1)
    kappa, beta = _fields(spec)
    ids = np.arange(spec.N, dtype=np.int64).reshape(spec.dims)
    diag = np.zeros(spec.dims)
    R, C, V = [], [], []
    for ax in range(d):
        lo = tuple(slice(0, n - 1) if a == ax else slice(None) for a in range(d))
        hi = tuple(slice(1, n) if a == ax else slice(None) for a in range(d))
        ka, kb = kappa[lo], kappa[hi]
        face = 2.0 * ka * kb / (ka + kb) / (h * h)
        diag[lo] += face
        diag[hi] += face
        for end in (0, n - 1):
            sl = tuple(end if a == ax else slice(None) for a in range(d))
            diag[sl] += kappa[sl] / (h * h)
        b = beta[..., ax] / h
        pos = np.maximum(b, 0.0)
        neg = np.minimum(b, 0.0)
        diag += pos - neg
        # node hi looks back at node lo when its beta is positive
        w_hi = -face - pos[hi]
        # node lo looks forward at node hi when its beta is negative
        e_lo = -face + neg[lo]
        R += [ids[hi].ravel(), ids[lo].ravel()]
        C += [ids[lo].ravel(), ids[hi].ravel()]
        V += [w_hi.ravel(), e_lo.ravel()]
    R.append(ids.ravel())
    C.append(ids.ravel())
    V.append(diag.ravel())
    return SparseMat.from_triplets(spec.N, spec.N, np.concatenate(R),
                                   np.concatenate(C), np.concatenate(V))


def default_levels(N):
    """ceil(log2(N/64)) — same rule as the reference (`problems.py:263-265`)."""
    return max(1, math.ceil(math.log(N / 64.0) / math.log(2.0)))


# ------------------------------------------------------------------ configs
# BASELINE.json "configs" (C2 is a kernel micro-benchmark, see bench.py)
CONFIGS = {
    "C1": dict(spec=UpwindSpec(n=64, ndim=2, beta_const=(20.0, 20.0)),
               levels=6, eps=1e-2, rhs_seed=0, tol=1e-12),
    "C3": dict(spec=UpwindSpec(n=256, ndim=2, kappa="loguniform", beta="uniform",
                               beta_range=50.0, seed=0),
               levels=10, eps=1e-3, rhs_seed=0, tol=1e-12),
    "C4": dict(spec=UpwindSpec(n=32, ndim=3, beta_const=(10.0, 10.0, 10.0)),
               levels=9, eps=1e-2, rhs_seed=1, tol=1e-12),
    "C5": dict(spec=UpwindSpec(n=64, ndim=3, kappa="loguniform", beta="uniform",
                               beta_range=20.0, seed=0),
               levels=11, eps=1e-2, rhs_seed=0, tol=1e-10),
}


def make_config(name, n=None, levels=None):
    """(A, dims, L, eps, b, tol) for a named config; `n` shrinks the grid
    (levels default to ceil(log2(N/64)) then) for fast parity cases."""
    cfg = CONFIGS[name]
    spec = cfg["spec"]
    if n is not None:
        spec = UpwindSpec(**{**spec.__dict__, "n": n})
    L = levels or (cfg["levels"] if n is None else default_levels(spec.N))
    A = upwind_convection_diffusion(spec)
    b = np.random.default_rng(cfg["rhs_seed"]).standard_normal(spec.N)
    return A, spec.dims, L, cfg["eps"], b, cfg["tol"]
