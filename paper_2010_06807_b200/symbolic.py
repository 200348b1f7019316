"""Symbolic (drop-free) fill prediction of the level driver.

`symbolic_fill_levels(A, tree)` mirrors the reference audit of the same name
(`pkg/src/nestqr/factor.py:1004-1050`): for every level, the set of
(row cluster, column cluster) block keys that can exist right after that
level's eliminations and before its merge, when nothing is dropped.  The
numeric driver must create blocks only inside it (reference test
`tests/test_factor.py:168-183`; here `tests/test_gpu_factor.py::
test_fill_within_symbolic_prediction` through `_StateView.trailing_keys`).

Eliminating cluster s couples every row cluster that holds a block in
column s -- plus s itself -- with every column cluster those rows touch
(`factor_interior`, factor.py:417-480); row and column s then disappear.
The device planner's predicted row flags (runtime.cu `predict_*`) are the
per-row refinement of this per-block rule, verified on the device.
"""
from __future__ import annotations

import numpy as np

from .sparse import as_csc


def symbolic_fill_levels(A, tree):
    """{level: set of (row cid, col cid)}: pattern after the level's
    eliminations, before its merge."""
    n, m, indptr, indices, data = as_csc(A)
    leaves = tree.leaf_clusters()
    col_owner = np.empty(tree.N, np.int64)
    row_owner = np.empty(tree.N, np.int64)
    for c in leaves:
        col_owner[np.asarray(c.cols)] = c.id
        row_owner[np.asarray(c.cols if c.rows is None else c.rows)] = c.id
    cols_of_entries = np.repeat(np.arange(n), np.diff(indptr))
    keys = np.unique(np.stack([row_owner[indices], col_owner[cols_of_entries]], axis=1), axis=0)
    by_row, by_col = {}, {}

    def link(i, j):
        by_row.setdefault(i, set()).add(j)
        by_col.setdefault(j, set()).add(i)

    for i, j in keys.tolist():
        link(i, j)
    out = {}
    for lev in range(tree.L, 0, -1):
        for c in tree.factor_at(lev):
            s = c.id
            panel_rows = set(by_col.get(s, ())) | {s}
            targets = set()
            for r in panel_rows:
                targets |= by_row.get(r, set())
            targets.discard(s)
            for r in panel_rows - {s}:
                for t in targets:
                    link(r, t)
            for r in by_col.pop(s, set()):        # column s leaves
                by_row[r].discard(s)
            for t in by_row.pop(s, set()):        # row s leaves
                if t in by_col:
                    by_col[t].discard(s)
        out[lev] = {(i, j) for i, js in by_row.items() for j in js}
        if lev >= 2:
            parent = {k: P.id for P in tree.active_at(lev - 1) for k in P.children}
            merged = {(parent[i], parent[j]) for i, js in by_row.items() for j in js}
            by_row, by_col = {}, {}
            for i, j in merged:
                link(i, j)
    return out
