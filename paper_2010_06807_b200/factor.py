"""Host level driver + device Factorization (drop-in for `nestqr.factor`).

``factorize`` keeps the reference's level loop verbatim in structure
(`pkg/src/nestqr/factor.py:771-911`): levels L..1; factor every cluster born
at the level in ascending id; once more than ``skip`` levels ran (and
lev >= 2), scale then sparsify every pending fragment with at least
``sparsify_min`` columns, in ascending id; merge fragments one depth up.
Each level operation is ONE call into the native library
(``include/spaqr_b200.h``), which owns the HBM-resident block store and runs
the hand-written sm_100a kernels; nothing numeric happens on the host.

``Factorization`` exposes what the reference's GMRES and tests use: ``N``,
``apply_qt``, ``solve_w``, ``apply_w`` (host arrays in / out, chains run on
the device), ``stats``, ``payload_scalars``, ``row_of_col``, ``options``,
``tree``, ``A`` and host views of the transform records (``q_chain`` /
``w_chain``) fetched lazily from device memory.
"""

from __future__ import annotations

import time

import numpy as np

from ._lib import Context
from .errors import DeviceError, NestqrError, SpeculationError
from .sparse import as_csc

MODES = ("scaled", "unscaled", "variant1", "variant2")


# --------------------------------------------------------------- record views

class HouseholderPanel:
    """Compact WY panel H = I - V T V^T (reference `kernels/__init__.py:73-118`)."""

    def __init__(self, V, tau, T, rows=None):
        self.V, self.tau, self.T, self.rows = V, tau, T, rows

    @property
    def m(self):
        return self.V.shape[0]

    @property
    def k(self):
        return self.V.shape[1]

    @property
    def payload_scalars(self):
        return self.V.size + self.tau.size + self.T.size


class _RecordView:
    kind = 0

    def __init__(self, F, idx, info):
        # the context, not the Factorization: no reference cycle, so the
        # device memory is released as soon as the last user drops F
        self._ctx, self._idx = F._ctx, idx
        self._m, self._k, self._n, self._rank = (int(x) for x in info[1:5])
        self.cid = int(info[5])          # cluster eliminated / scaled / compressed
        self._unscaled, self._f = bool(info[6]), int(info[7])
        self._cache = {}

    def _get(self, which):
        if which in self._cache:
            return self._cache[which]
        ctx = self._ctx
        m, k, n = self._m, self._k, self._n
        if which in (0, 1, 2):
            size = {0: m, 1: self._ncols(), 2: self._ncolsn()}[which]
            out = np.empty(size, np.int64)
        elif which == 3:
            out = np.empty((k, m))
        elif which == 4:
            out = np.empty(k)
        elif which in (5, 6):
            out = np.empty((k, k))
        else:
            out = np.empty((n, k))
        if out.size:
            ctx.call("spq_record_get", self._idx, which, out.ctypes.data)
        if which == 3 or which in (5, 6, 7):
            out = np.ascontiguousarray(out.T)     # device storage is column-major
        self._cache[which] = out
        return out

    def _ncols(self):
        return self._k if self.kind == 1 else self._m

    def _ncolsn(self):
        return self._n

    @property
    def rows(self):
        return self._get(0)

    @property
    def panel(self):
        return HouseholderPanel(self._get(3), self._get(4), self._get(5), self.rows)


class BlockHouseholder(_RecordView):
    """Interior elimination record (reference `factor.py:78-113`)."""
    kind = 1

    cols_s = property(lambda s: s._get(1))
    cols_n = property(lambda s: s._get(2))
    R_ss = property(lambda s: s._get(6))
    R_sn = property(lambda s: s._get(7))

    @property
    def payload_scalars(self):
        return self._m * self._k + 3 * self._k * self._k + self._k + self._k * self._n


class InterfaceScaling(_RecordView):
    """Interface scaling record (reference `factor.py:116-142`)."""
    kind = 2

    cols = property(lambda s: s._get(1))
    R_pp = property(lambda s: s._get(6))

    @property
    def payload_scalars(self):
        return 3 * self._k * self._k + self._k


class Sparsifier(_RecordView):
    """Sparsifier record (reference `factor.py:145-205`): scaled flavour
    (Q panel only) or unscaled flavour (Q panel + H_f panel, R_ff, R_fc)."""
    kind = 3

    cols = property(lambda s: s._get(1))
    rank = property(lambda s: s._rank)

    @property
    def scaled(self):
        return not self._unscaled

    @property
    def fine(self):
        return self._m - self._rank

    @property
    def q_panel(self):
        return self.panel

    def _getu(self, which, shape):
        if which not in self._cache:
            out = np.empty(shape[::-1] if len(shape) == 2 else shape)
            if out.size:
                self._ctx.call("spq_record_get", self._idx, which, out.ctypes.data)
            self._cache[which] = np.ascontiguousarray(out.T) if len(shape) == 2 else out
        return self._cache[which]

    @property
    def hf_panel(self):
        if self.scaled:
            return None
        f, m = self._f, self._m
        return HouseholderPanel(self._getu(8, (m, f)), self._getu(9, (f,)),
                                self._getu(10, (f, f)), self.rows)

    @property
    def R_ff(self):
        return None if self.scaled else self._getu(6, (self._f, self._f))

    @property
    def R_fc(self):
        return None if self.scaled else self._getu(7, (self._f, self._rank))

    @property
    def payload_scalars(self):
        n = self._m * self._k + self._k + self._k * self._k
        if not self.scaled:
            f = self._f
            n += self._m * f + f + f * f + f * f + f * self._rank
        return n


class Permutation:
    def __init__(self, row_of_col):
        self.row_of_col = row_of_col

    payload_scalars = 0


class DiagonalScaling:
    """W-chain[0]; the scale vector itself stays on the device."""

    def __init__(self, N):
        self.N = N

    @property
    def payload_scalars(self):
        return self.N


_VIEW = {1: BlockHouseholder, 2: InterfaceScaling, 3: Sparsifier}


# ------------------------------------------------------------- factorization

class Factorization:
    def __init__(self, ctx, A, tree, row_of_col, stats, options, equilibrate):
        self._ctx = ctx
        self.A = A
        self.N = int(A.ncols)
        self.tree = tree
        self.row_of_col = row_of_col
        self.stats = stats
        self.options = options
        self._equil = equilibrate
        self._records = None

    # ---------------------------------------------------------- records
    def _recs(self):
        if self._records is None:
            n = self._ctx.lib.spq_num_records(self._ctx.h)
            recs = []
            info = np.zeros(8, np.int64)
            for i in range(n):
                self._ctx.call("spq_record_info", i, info)
                recs.append(_VIEW[int(info[0])](self, i, info.copy()))
            self._records = recs
        return self._records

    @property
    def q_chain(self):
        return self._recs() + [Permutation(self.row_of_col)]

    @property
    def w_chain(self):
        return ([DiagonalScaling(self.N)] if self._equil else []) + self._recs()

    @property
    def payload_scalars(self):
        return self._ctx.i64("spq_payload_scalars")

    # ---------------------------------------------------------- chains
    def _run(self, name, v):
        v = np.asarray(v, dtype=np.float64)
        if v.ndim == 0 or v.shape[0] != self.N:
            raise NestqrError(f"vector of length {v.shape[0] if v.ndim else 0} incompatible "
                              f"with matrix of size {self.N}")
        vec = v.ndim == 1
        X = v.reshape(self.N, -1)
        nrhs = X.shape[1]
        src = np.asfortranarray(X).ravel(order="F")
        out = np.empty_like(src)
        if nrhs:
            self._ctx.call(name, src, out, nrhs)
        out = out.reshape((self.N, nrhs), order="F")
        return out[:, 0].copy() if vec else np.ascontiguousarray(out)

    def apply_qt(self, b):
        """P^T Q^T b (reference `factor.py:281-286`)."""
        return self._run("spq_apply_qt_host", b)

    def apply_w(self, x):
        """W x (reference `factor.py:288-293`)."""
        return self._run("spq_apply_w_host", x)

    def solve_w(self, y):
        """W^{-1} y (reference `factor.py:295-300`)."""
        return self._run("spq_solve_w_host", y)

    def gmres_device(self, A, b, tol=1e-12, maxit=300, restart=None, x0=None):
        """GMRES of `solve.py:66-209` run entirely on the device (spq_gmres);
        returns (x, iterations, history, converged, best_residual)."""
        import ctypes as C
        from .sparse import as_csc
        n, m, indptr, indices, data = as_csc(A)
        if n != self.N or m != self.N:
            raise NestqrError("factorization size does not match the matrix")
        # uploaded on every call: a cache keyed on the matrix object would go
        # stale when a matrix is edited in place or its id is reused (the
        # CSR upload costs ~1 ms at C3 against tens of ms of iterations)
        self._ctx.call("spq_set_matrix", n, indptr, indices, data)
        b = np.ascontiguousarray(b, dtype=np.float64)
        x = np.empty(n)
        hist = np.empty(max(int(maxit), 0) + 1)
        its, conv, best = C.c_int(), C.c_int(), C.c_double()
        x0a = None if x0 is None else np.ascontiguousarray(x0, dtype=np.float64)
        self._ctx.call("spq_gmres", b, None if x0a is None else x0a.ctypes.data, float(tol),
                       int(maxit), 0 if restart is None else int(restart), x, hist,
                       C.byref(its), C.byref(conv), C.byref(best))
        k = int(its.value)
        nh = k + 1 if float(np.linalg.norm(b)) != 0.0 else 1
        return x, k, hist[:nh].copy(), bool(conv.value), float(best.value)

    def materialize_preconditioned(self):
        X = self.solve_w(np.eye(self.N))
        from .sparse import matvec
        return self.apply_qt(matvec(self.A, X))

    def materialize_w(self):
        return self.apply_w(np.eye(self.N))

    def stats_fieldnames(self):
        return list(self.stats[0].keys()) if self.stats else []

    def device_timings(self):
        return self._ctx.timings()


class _StateView:
    """What observer hooks see: live cluster sizes from the device store."""

    class _Sized:
        def __init__(self, ctx, axis):
            self.ctx, self.axis = ctx, axis

        def __getitem__(self, cid):
            import ctypes as C
            r, c = C.c_int64(), C.c_int64()
            self.ctx.call("spq_cluster_size", int(cid), C.byref(r), C.byref(c))
            return range(int(r.value if self.axis == 0 else c.value))

    def __init__(self, ctx):
        self.ctx = ctx
        self.rows_of = self._Sized(ctx, 0)
        self.cols_of = self._Sized(ctx, 1)

    def trailing_keys(self):
        """(row cluster, column cluster) of every live trailing block: the
        keys of the reference's `state.trailing` dict (factor.py:349)."""
        import ctypes as C
        n = C.c_int64()
        z = np.zeros(0, np.int32)
        self.ctx.call("spq_trailing_keys", 0, z, z, C.byref(n))
        r, c = np.zeros(n.value, np.int32), np.zeros(n.value, np.int32)
        self.ctx.call("spq_trailing_keys", int(n.value), r, c, C.byref(n))
        return set(zip(r.tolist(), c.tolist()))


def _cluster_lists(clusters, attr):
    """CSR-style (ptr, values) of the clusters' row or column index lists
    (one concatenate: a per-cluster conversion loop cost ~2 ms per call at C3)."""
    vals = []
    for c in clusters:
        a = getattr(c, attr)
        vals.append(c.cols if a is None else a)
    ptr = np.zeros(len(vals) + 1, np.int64)
    if not vals:
        return ptr, np.zeros(0, np.int64)
    np.cumsum([len(a) for a in vals], out=ptr[1:])
    return ptr, np.concatenate(vals).astype(np.int64, copy=False)


def factorize(A, tree=None, eps=1e-3, **kw):
    """Run the multilevel factorization on the B200 (signature of the reference
    `factorize`, `factor.py:771-803`).

    Device memory of contexts that are unreachable but not yet collected
    (reference cycles) is only returned when the garbage collector runs: on an
    out-of-memory failure the context is released, garbage is collected and
    the factorization runs once more."""
    try:
        return _factorize_spec(A, tree, eps, **kw)
    except DeviceError as e:
        if "out of memory" not in str(e):
            raise
    import gc
    gc.collect()
    return _factorize_spec(A, tree, eps, **kw)


def _factorize_spec(A, tree, eps, **kw):
    """A predicted row-nonzero flag that the device finds wrong (an exact
    cancellation the symbolic rules cannot see) surfaces as SpeculationError
    at the next synchronisation point, anywhere in the level loop: redo the
    factorization with flags read back exactly.  The failed attempt's device
    time stays in the measured total."""
    held = {}
    try:
        return _factorize(A, tree, eps, _held=held, **kw)
    except SpeculationError:
        if not kw.get("_speculate", True):
            raise
    ctx = held.get("ctx")
    lost_ms = 0.0
    if ctx is not None:
        if kw.get("_marks"):
            import ctypes as C
            ms = C.c_float()
            ctx.call("spq_mark", 1)
            ctx.call("spq_synchronize")
            ctx.call("spq_mark_elapsed", 0, 1, C.byref(ms))
            lost_ms = float(ms.value)
        ctx.close()
    kw = dict(kw, _speculate=False)
    F = _factorize(A, tree, eps, **kw)
    F.spec_retries = 1
    if F.device_ms is not None:
        F.device_ms += lost_ms
    return F


def _factorize(A, tree=None, eps=1e-3, *, levels=None, sparsify=True, scaling=True,
               scale_every=1, skip=2, sparsify_min=40, mode="scaled",
               row_heuristic="same-as-columns", equilibrate=True, observer=None, device=0,
               _marks=False, _memstats=False, _speculate=True, _held=None):
    if mode not in MODES:
        raise NestqrError(f"unknown sparsification mode {mode!r}")
    if mode == "unscaled":
        scaling = False
    if int(scale_every) < 1:
        raise NestqrError(f"scale_every must be >= 1, got {scale_every}")
    mode_id = MODES.index(mode)
    if tree is None:
        raise NestqrError("the B200 path needs a cluster tree (e.g. ordering.partition_geometric)")
    n, m, indptr, indices, data = as_csc(A)
    if n != m:
        raise NestqrError(f"matrix must be square, got {(n, m)}")
    leaves = tree.leaf_clusters()
    if leaves and leaves[0].rows is None:
        if row_heuristic not in ("same-as-columns", "cols"):
            raise NestqrError(f"row heuristic {row_heuristic!r} not available on the B200 path")
        from .ordering import assign_rows_same_as_columns
        assign_rows_same_as_columns(tree)
    L = tree.L
    ctx = Context(device)
    if _held is not None:
        _held["ctx"] = ctx
    if not _speculate:
        ctx.call("spq_set_option", b"speculate", 0)
    leaf_ids = np.array([c.id for c in leaves], np.int32)
    rptr, rows = _cluster_lists(leaves, "rows")
    cptr, cols = _cluster_lists(leaves, "cols")
    if _marks:
        # the device-timed region opens BEFORE the load: equilibration and the
        # CSC -> block scatter are part of the reference's factorize
        # (TrailingState.__init__, factor.py:328-374)
        ctx.call("spq_mark", 0)
    ctx.call("spq_load", n, indptr, indices, data, int(bool(equilibrate)),
             len(tree.clusters), len(leaves), leaf_ids, rptr, rows, cptr, cols)

    import ctypes as C

    def size_of(cid):
        r, c = C.c_int64(), C.c_int64()
        ctx.call("spq_cluster_size", int(cid), C.byref(r), C.byref(c))
        return int(c.value)

    def sizes_of(ids):
        ids = np.asarray(ids, np.int32)
        out = np.zeros(len(ids), np.int64)
        if len(ids):
            ctx.call("spq_cluster_sizes", len(ids), ids, out)
        return out

    state = _StateView(ctx)
    stats = []
    ranks_log = []
    by_level = {lev: sorted(c.id for c in tree.factor_at(lev)) for lev in range(1, L + 1)}
    pending = {lev: sorted(c.id for c in tree.sparsify_at(lev)) for lev in range(1, L + 1)}
    n_sparsified_levels = 0
    for lev in range(L, 0, -1):
        st = {"level": lev, "cols_before": ctx.i64("spq_total_cols"),
              "n_factored": 0, "factored_cols": 0,
              "n_scaled": 0, "n_sparsified": 0, "fine_retired": 0,
              "dropped_max": 0.0,
              "iface_q1": 0.0, "iface_q2": 0.0, "iface_q3": 0.0,
              "iface_max": 0, "cols_after": 0,
              "trailing_nnz": 0, "trailing_blocks": 0,
              "t_factor": 0.0, "t_scale": 0.0, "t_sparsify": 0.0, "t_merge": 0.0}
        t0 = time.perf_counter()
        ids = by_level[lev]
        st["factored_cols"] = int(sizes_of(ids).sum())
        if ids:
            ctx.call("spq_factor", len(ids), np.asarray(ids, np.int32))
        st["n_factored"] = len(ids)
        st["t_factor"] = time.perf_counter() - t0

        run_sparsify = sparsify and (L - lev + 1) > skip and lev >= 2 and pending[lev]
        if run_sparsify:
            n_sparsified_levels += 1
            psz = sizes_of(pending[lev])
            todo = [p for p, z in zip(pending[lev], psz) if z >= sparsify_min]
            # scaling on every scale_every-th sparsified level (factor.py:847-861)
            do_scale = bool(scaling) and (n_sparsified_levels - 1) % int(scale_every) == 0
            if todo:
                ids_t = np.asarray(todo, np.int32)
                if do_scale:
                    t0 = time.perf_counter()
                    done = np.zeros(len(todo), np.int32)
                    ctx.call("spq_scale", len(todo), ids_t, done)
                    st["n_scaled"] = int(done.sum())
                    st["t_scale"] = time.perf_counter() - t0
                on_sp = getattr(observer, "on_sparsify", None)
                t0 = time.perf_counter()
                rank = np.zeros(len(todo), np.int32)
                before = np.zeros(len(todo), np.int32)
                dropped = np.zeros(len(todo))
                done = np.zeros(len(todo), np.int32)
                if on_sp is None:
                    ctx.call("spq_sparsify_ex", len(todo), ids_t, float(eps), mode_id,
                             int(do_scale), rank, before, dropped, done)
                else:
                    for t, p in enumerate(todo):
                        on_sp(state, p, "before")
                        r1, b1 = np.zeros(1, np.int32), np.zeros(1, np.int32)
                        d1, k1 = np.zeros(1), np.zeros(1, np.int32)
                        ctx.call("spq_sparsify_ex", 1, ids_t[t:t + 1], float(eps), mode_id,
                                 int(do_scale), r1, b1, d1, k1)
                        rank[t], before[t], dropped[t], done[t] = r1[0], b1[0], d1[0], k1[0]
                        on_sp(state, p, "after")
                for t in range(len(todo)):
                    if done[t]:
                        st["n_sparsified"] += 1
                        st["fine_retired"] += int(before[t] - rank[t])
                        st["dropped_max"] = max(st["dropped_max"], float(dropped[t]))
                st["t_sparsify"] = time.perf_counter() - t0
                ranks_log.extend((lev, int(p), int(b), int(r)) for p, b, r in zip(todo, before, rank))

        sizes = [int(z) for z in sizes_of(pending[lev])]
        if sizes:
            q1, q2, q3 = np.percentile(sizes, [25, 50, 75])
            st["iface_q1"], st["iface_q2"], st["iface_q3"] = float(q1), float(q2), float(q3)
            st["iface_max"] = int(max(sizes))
        st["cols_after"] = ctx.i64("spq_total_cols")
        nb = C.c_int64()
        on_lv = getattr(observer, "on_level", None)
        if on_lv is None:   # nnz read once after the last level (no per-level sync)
            ctx.call("spq_trailing_stats_async", len(stats), C.byref(nb))
        else:
            nz = C.c_int64()
            ctx.call("spq_trailing_stats", C.byref(nb), C.byref(nz))
            st["trailing_nnz"] = int(nz.value)
        st["trailing_blocks"] = int(nb.value)
        if _memstats:
            h = ctx.timings()["host"]
            st["_live_gb"], st["_peak_gb"] = h["live_bytes"] / 1e9, h["peak_bytes"] / 1e9
        if on_lv is not None:
            on_lv(state, lev, st)
        if lev >= 2:
            t0 = time.perf_counter()
            parents = tree.active_at(lev - 1)
            pid = np.asarray([P.id for P in parents], np.int32)
            cptr_m = np.zeros(len(parents) + 1, np.int32)
            kids = []
            for i, P in enumerate(parents):
                kids.extend(P.children)
                cptr_m[i + 1] = len(kids)
            ctx.call("spq_merge", len(parents), pid, cptr_m, np.asarray(kids, np.int32))
            st["t_merge"] = time.perf_counter() - t0
        stats.append(st)

    ctx.call("spq_finish")
    if getattr(observer, "on_level", None) is None and stats:
        nnz = np.zeros(len(stats), np.int64)
        ctx.call("spq_trailing_nnz", len(stats), nnz)
        for st, z in zip(stats, nnz):
            st["trailing_nnz"] = int(z)
    device_ms = None
    if _marks:
        ctx.call("spq_mark", 1)
        ms = C.c_float()
        ctx.call("spq_mark_elapsed", 0, 1, C.byref(ms))
        device_ms = float(ms.value)
    roc = np.empty(n, np.int64)
    ctx.call("spq_row_of_col", roc)
    options = {"eps": eps, "mode": mode, "sparsify": sparsify, "scaling": scaling,
               "scale_every": scale_every, "skip": skip, "sparsify_min": sparsify_min,
               "row_heuristic": row_heuristic, "equilibrate": equilibrate, "levels": L}
    F = Factorization(ctx, A, tree, roc, stats, options, equilibrate)
    F.sparsify_log = ranks_log   # (level, interface, |cols| before, accepted rank)
    F.device_ms = device_ms      # load start -> finish on the library stream (bench)
    F.spec_retries = 0
    return F
