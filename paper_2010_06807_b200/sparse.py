"""Compressed-sparse-column input container.

The factorization accepts any object exposing ``nrows, ncols, indptr,
indices, data`` (CSC, row indices increasing within a column) — in
particular the reference's own ``nestqr.sparse.SparseMat``
(`pkg/src/nestqr/sparse.py:15-138`).  This class is the minimal stand-in
used when the reference package is not installed (e.g. on the GPU box):
triplet assembly sums duplicates and keeps explicit zeros, exactly as the
reference's ``from_triplets`` (`sparse.py:40-65`) does, because stored zeros
change nothing numerically but do change the block structure the driver
builds.
"""

from __future__ import annotations

import numpy as np

from .errors import NestqrError


class SparseMat:
    __slots__ = ("nrows", "ncols", "indptr", "indices", "data")

    def __init__(self, nrows, ncols, indptr, indices, data):
        self.nrows = int(nrows)
        self.ncols = int(ncols)
        self.indptr = np.asarray(indptr, dtype=np.int64)
        self.indices = np.asarray(indices, dtype=np.int64)
        self.data = np.asarray(data, dtype=np.float64)

    @classmethod
    def from_triplets(cls, nrows, ncols, rows, cols, vals):
        rows = np.asarray(rows, dtype=np.int64)
        cols = np.asarray(cols, dtype=np.int64)
        vals = np.asarray(vals, dtype=np.float64)
        if rows.size and (rows.min() < 0 or rows.max() >= nrows
                          or cols.min() < 0 or cols.max() >= ncols):
            raise NestqrError("triplet index out of range")
        key = cols * np.int64(nrows) + rows
        order = np.argsort(key, kind="stable")
        key, vals = key[order], vals[order]
        if key.size:
            first = np.r_[True, key[1:] != key[:-1]]
            grp = np.cumsum(first) - 1
            summed = np.zeros(int(grp[-1]) + 1)
            np.add.at(summed, grp, vals)
            key, vals = key[first], summed
        c = key // nrows
        r = key - c * nrows
        indptr = np.zeros(ncols + 1, dtype=np.int64)
        np.cumsum(np.bincount(c, minlength=ncols), out=indptr[1:])
        return cls(nrows, ncols, indptr, r, vals)

    @classmethod
    def from_dense(cls, D):
        D = np.asarray(D, dtype=np.float64)
        r, c = np.nonzero(D)
        return cls.from_triplets(D.shape[0], D.shape[1], r, c, D[r, c])

    @classmethod
    def identity(cls, n):
        ar = np.arange(n, dtype=np.int64)
        return cls(n, n, np.arange(n + 1, dtype=np.int64), ar, np.ones(n))

    @property
    def nnz(self):
        return int(self.indptr[-1])

    @property
    def shape(self):
        return (self.nrows, self.ncols)

    def to_scipy(self):
        from scipy.sparse import csc_matrix
        return csc_matrix((self.data, self.indices, self.indptr),
                          shape=(self.nrows, self.ncols))

    def to_dense(self):
        return self.to_scipy().toarray()

    def to_triplets(self):
        cols = np.repeat(np.arange(self.ncols, dtype=np.int64), np.diff(self.indptr))
        return self.indices.copy(), cols, self.data.copy()

    def matvec(self, x):
        return self.to_scipy() @ np.asarray(x, dtype=np.float64)

    def __matmul__(self, x):
        return self.matvec(x)


def as_csc(A):
    """Normalise a duck-typed CSC matrix into contiguous int64/float64 arrays."""
    for attr in ("nrows", "ncols", "indptr", "indices", "data"):
        if not hasattr(A, attr):
            raise NestqrError(f"matrix object lacks CSC attribute {attr!r}")
    return (int(A.nrows), int(A.ncols),
            np.ascontiguousarray(A.indptr, dtype=np.int64),
            np.ascontiguousarray(A.indices, dtype=np.int64),
            np.ascontiguousarray(A.data, dtype=np.float64))


def matvec(A, x):
    """Host CSC product used by the GMRES wrapper (the reference keeps the
    matvec on the host too, `sparse.py:110-113`)."""
    if hasattr(A, "matvec"):
        return A.matvec(x)
    n, m, p, i, d = as_csc(A)
    from scipy.sparse import csc_matrix
    return csc_matrix((d, i, p), shape=(n, m)) @ x
