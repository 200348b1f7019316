"""Geometric nested-dissection cluster hierarchy (host side).

The north star keeps the ordering on the host; this module exists so the
B200 path can run where the reference package is not installed.  It builds
the SAME tree as the reference's ``partition_geometric``
(`pkg/src/nestqr/ordering.py:398-419`, engine `_build_tree` `:212-275`,
cutter `_GeoCutter` `:319-395`, id assignment `_assemble` `:278-313`):
cluster ids decide the driver's processing order, so the tests
pin this restatement against the reference's trees by hash
(`tests/golden/trees.json`).

Any object with the reference ``ClusterTree`` attributes (``N, L, clusters,
depth_ids, active_at, factor_at, sparsify_at, leaf_clusters``) is accepted
by ``factorize`` — including the reference's own trees.

Construction, restated:

* boxes are cut level-synchronously; the cut plane pair {m, m+1} lies
  across the first longest axis with m = lo + (extent-1)//2;
* each separator exists whole at its birth depth and, one depth further
  down per round, is refined by every new cut whose region box lies within
  an L1 gap of 2 of the fragment's box (three bands along the cut axis);
* ids: leaf interiors first (final region order), then for each separator
  in birth order, its fragments depth by depth.
"""

from __future__ import annotations

import numpy as np

from .errors import NestqrError, PartitionError

KIND_INTERIOR = "interior"
KIND_INTERFACE = "interface"


class Cluster:
    __slots__ = ("id", "kind", "level", "depth", "sep", "cols", "rows",
                 "parent", "children", "neighbors")

    def __init__(self, id, kind, level, depth, sep, cols, rows=None,
                 parent=-1, children=None):
        self.id, self.kind, self.level, self.depth, self.sep = id, kind, level, depth, sep
        self.cols = cols
        self.rows = rows
        self.parent = parent
        self.children = children if children is not None else []
        self.neighbors = []

    @property
    def size(self):
        return len(self.cols)


class ClusterTree:
    def __init__(self, N, L, clusters, depth_ids, meta=None):
        self.N, self.L = N, L
        self.clusters = clusters
        self.depth_ids = depth_ids
        self.meta = meta or {}

    def cluster(self, cid):
        return self.clusters[cid]

    def active_at(self, depth):
        return [self.clusters[i] for i in self.depth_ids[depth]]

    def factor_at(self, level):
        return [c for c in self.active_at(level) if c.level == level]

    def sparsify_at(self, level):
        return [c for c in self.active_at(level) if c.level < level]

    def leaf_clusters(self):
        return self.active_at(self.L)


def _box_ids(lo, hi, strides):
    if (hi < lo).any():
        return np.empty(0, np.int64)
    axes = [np.arange(a, b + 1, dtype=np.int64) * s for a, b, s in zip(lo, hi, strides)]
    flat = axes[0]
    for ax in axes[1:]:
        flat = (flat[:, None] + ax[None, :]).ravel()
    return flat


def partition_geometric(dims, L):
    dims = tuple(int(d) for d in dims)
    if any(d < 1 for d in dims):
        raise NestqrError(f"bad grid dims {dims}")
    L = int(L)
    if L < 1:
        raise PartitionError(f"level count must be >= 1, got {L}")
    nd = len(dims)
    N = int(np.prod(dims))
    strides = np.array([int(np.prod(dims[a + 1:])) for a in range(nd)], np.int64)

    regions = [(np.zeros(nd, np.int64), np.array(dims, np.int64) - 1)]
    # fragment = [sep id, node ids, box lo, box hi]
    frags = []
    birth = []                # birth[sep] = level
    snaps = {}                # (sep, depth) -> [node arrays]

    for t in range(1, L):
        cuts = []             # (region lo, region hi, axis, m)
        nxt = []
        for lo, hi in regions:
            ext = hi - lo + 1
            ax = int(np.argmax(ext))
            if ext[ax] < 4:
                raise PartitionError(f"grid box extent {tuple(int(e) for e in ext)} "
                                     f"too small for a two-plane cut")
            m = int(lo[ax] + (ext[ax] - 1) // 2)
            s_lo, s_hi = lo.copy(), hi.copy()
            s_lo[ax], s_hi[ax] = m, m + 1
            l_hi = hi.copy()
            l_hi[ax] = m - 1
            r_lo = lo.copy()
            r_lo[ax] = m + 2
            if l_hi[ax] < lo[ax] or r_lo[ax] > hi[ax]:
                raise PartitionError(f"level count {L} too deep for region {tuple(ext)}")
            nxt += [(lo.copy(), l_hi), (r_lo, hi.copy())]
            cuts.append((lo, hi, ax, m))
            sep_nodes = _box_ids(s_lo, s_hi, strides)
            if len(sep_nodes):
                birth.append(t)
                frags.append([len(birth) - 1, sep_nodes, s_lo, s_hi])
        refined = []
        for f in frags:
            if birth[f[0]] == t:
                refined.append(f)
                continue
            parts = [f]
            for rlo, rhi, ax, m in cuts:
                gap = np.maximum(0, np.maximum(rlo - f[3], f[2] - rhi))
                if int(gap.sum()) > 2:
                    continue
                split = []
                for q in parts:
                    coord = (q[1] // strides[ax]) % dims[ax]
                    bands = []
                    for b0, b1 in ((q[2][ax], m - 1), (m, m + 1), (m + 2, q[3][ax])):
                        b0, b1 = max(b0, int(q[2][ax])), min(b1, int(q[3][ax]))
                        if b0 > b1:
                            continue
                        sel = (coord >= b0) & (coord <= b1)
                        if sel.any():
                            qlo, qhi = q[2].copy(), q[3].copy()
                            qlo[ax], qhi[ax] = b0, b1
                            bands.append([q[0], q[1][sel], qlo, qhi])
                    split += [q] if len(bands) == 1 else bands
                parts = split
            refined += parts
        frags = refined
        for f in frags:
            snaps.setdefault((f[0], t), []).append(f[1])
        regions = nxt
    for f in frags:
        snaps.setdefault((f[0], L), []).append(f[1])

    clusters = []
    depth_ids = {d: [] for d in range(1, L + 1)}

    def add(kind, level, depth, sep, cols):
        c = Cluster(len(clusters), kind, level, depth, sep, np.sort(cols).astype(np.int64))
        clusters.append(c)
        depth_ids[depth].append(c.id)
        return c.id

    for lo, hi in regions:
        add(KIND_INTERIOR, L, L, -1, _box_ids(lo, hi, strides))
    owner = np.full(N, -1, np.int64)
    for s, lvl in enumerate(birth):
        prev = []
        for d in range(lvl, L + 1):
            cur = [add(KIND_INTERFACE, lvl, d, s, nodes) for nodes in snaps.get((s, d), [])]
            if prev:
                for p in prev:
                    owner[clusters[p].cols] = p
                for c in cur:
                    p = int(owner[clusters[c].cols[0]])
                    clusters[c].parent = p
                    clusters[p].children.append(c)
            prev = cur
    tree = ClusterTree(N, L, clusters, depth_ids, meta={"kind": "geometric", "dims": list(dims)})
    assign_rows_same_as_columns(tree)
    return tree


def assign_rows_same_as_columns(tree):
    """Row i joins the cluster owning column i (the reference default,
    `ordering.py:681-724`, heuristic 'same-as-columns'); unions propagate
    up the merge hierarchy so every diagonal block is square."""
    for c in tree.leaf_clusters():
        c.rows = c.cols.copy()
    for d in range(tree.L - 1, 0, -1):
        for c in tree.active_at(d):
            if not c.children:
                raise PartitionError(f"cluster {c.id} at depth {d} has no children")
            c.rows = np.sort(np.concatenate([tree.cluster(k).rows for k in c.children]))


def tree_digest(tree):
    """sha256 over (id, kind, level, depth, parent, children, cols) of every
    cluster and the depth lists — pins this tree against the reference's."""
    import hashlib
    h = hashlib.sha256()
    h.update(np.int64([tree.N, tree.L]).tobytes())
    for c in tree.clusters:
        h.update(f"{c.id}|{c.kind}|{c.level}|{c.depth}|{c.parent}|{list(c.children)}|".encode())
        h.update(np.asarray(c.cols, np.int64).tobytes())
    for d in sorted(tree.depth_ids):
        h.update(np.int64(list(tree.depth_ids[d])).tobytes())
    return h.hexdigest()
