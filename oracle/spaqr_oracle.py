"""TEST INFRASTRUCTURE ONLY — numpy restatement of the reference spaQR path.

See ``oracle/__init__.py`` for who may import this.  Each function cites the
reference lines (relative to ``/root/reference/pkg/src/nestqr``) whose
semantics it restates; the restatement is pinned against the live reference
through ``tests/golden`` (see ``tests/test_oracle.py``).

Layout: dense blocks are C-ordered numpy arrays keyed (row cluster, col
cluster) in a dict, exactly the reference's block model
(`factor.py:320-392`); all arithmetic is float64.
"""

from __future__ import annotations

import math

import numpy as np

PIVOT_FLOOR = 1e-14          # kernels/__init__.py:70


class OracleError(Exception):
    pass


class OracleSingularPivot(OracleError):
    def __init__(self, index, value, context=""):
        super().__init__(f"singular pivot in {context}: |R[{index},{index}]| = {abs(value):.3e}")
        self.index, self.value, self.context = index, value, context


# =============================================================== dense kernels

def reflector(x):
    """Householder vector with v0 = 1, the reference convention
    (`kernels/_numba.py:14-35`): beta = +||x||, v0 = alpha - beta when
    alpha <= 0 else -sigma/(alpha+beta); sigma == 0 gives tau = 0 (alpha >= 0)
    or tau = 2 with beta = -alpha.  Returns (v, tau, beta)."""
    alpha = float(x[0])
    tail = x[1:]
    sigma = float(tail @ tail)
    v = np.empty(len(x))
    v[0] = 1.0
    if sigma == 0.0:
        v[1:] = 0.0
        return (v, 0.0, alpha) if alpha >= 0.0 else (v, 2.0, -alpha)
    beta = math.sqrt(alpha * alpha + sigma)
    v0 = alpha - beta if alpha <= 0.0 else -sigma / (alpha + beta)
    v[1:] = tail / v0
    return v, -v0 / beta, beta


def larft(V, tau):
    """Forward/columnwise compact-WY T with H_1..H_k = I - V T V^T
    (`kernels/_numba.py:101-117`)."""
    k = V.shape[1]
    T = np.zeros((k, k))
    G = V.T @ V
    for i in range(k):
        T[i, i] = tau[i]
        if i and tau[i] != 0.0:
            T[:i, i] = -tau[i] * (T[:i, :i] @ G[:i, i])
    return T


def house_qr(B, nb=32):
    """Blocked Householder QR, m >= k (`kernels/_numba.py:52-84`): nb-column
    panels factored column by column, trailing columns updated with the
    panel's compact WY.  Returns V (m x k, unit lower trapezoidal), tau, R
    (k x k, diag >= 0)."""
    W = np.array(B, dtype=np.float64, copy=True)
    m, k = W.shape
    V = np.zeros((m, k))
    tau = np.zeros(k)
    for j0 in range(0, k, nb):
        j1 = min(j0 + nb, k)
        for j in range(j0, j1):
            v, t, beta = reflector(W[j:, j])
            V[j:, j] = v
            tau[j] = t
            if t != 0.0 and j + 1 < j1:
                W[j:, j + 1:j1] -= np.outer(t * v, v @ W[j:, j + 1:j1])
            W[j, j] = beta
            W[j + 1:, j] = 0.0
        if j1 < k:
            Vb = V[j0:, j0:j1]
            Tb = larft(Vb, tau[j0:j1])
            W[j0:, j1:] -= Vb @ (Tb.T @ (Vb.T @ W[j0:, j1:]))
    return V, tau, np.triu(W[:k, :k])


def wy_apply(V, T, C, transpose):
    """C - V T^T V^T C (transpose) or C - V T V^T C (`kernels/__init__.py:100-118`)."""
    if V.shape[1] == 0:
        return np.array(C, dtype=np.float64, copy=True)
    Tm = T.T if transpose else T
    return C - V @ (Tm @ (V.T @ C))


def cpqr_threshold(M, eps, min_rank=0):
    """Threshold column-pivoted QR with early stop (`kernels/_numba.py:120-167`):
    trailing column norms recomputed every step, first index wins ties,
    stop at step i >= 1 once max norm < eps * norm0 (and i >= min_rank).
    Returns (V[:, :r], tau[:r], Tred, perm, r)."""
    T = np.array(M, dtype=np.float64, copy=True)
    m, k = T.shape
    kmax = min(m, k)
    perm = np.arange(k, dtype=np.int64)
    V = np.zeros((m, kmax))
    tau = np.zeros(kmax)
    norm0 = 0.0
    r = kmax
    for i in range(kmax):
        sub = T[i:, i:]
        nrms = np.sqrt(np.einsum("ij,ij->j", sub, sub))
        p = i + int(np.argmax(nrms))
        nrm = float(nrms[p - i])
        if i == 0:
            norm0 = nrm
            if norm0 == 0.0:
                r = 0
                break
        elif nrm < eps * norm0 and i >= min_rank:
            r = i
            break
        if p != i:
            T[:, [i, p]] = T[:, [p, i]]
            perm[[i, p]] = perm[[p, i]]
        v, t, beta = reflector(T[i:, i])
        V[i:, i] = v
        tau[i] = t
        if t != 0.0 and i + 1 < k:
            T[i:, i + 1:] -= np.outer(t * v, v @ T[i:, i + 1:])
        T[i, i] = beta
        T[i + 1:, i] = 0.0
    return V[:, :r], tau[:r], T, perm, r


def rrqr_threshold(M, eps, min_rank=0):
    """(`kernels/__init__.py:174-199`) -> dict(V, tau, T, R, resid, perm, rank)."""
    if not (0.0 <= eps < 1.0):
        raise OracleError(f"eps out of range: {eps}")
    M = np.ascontiguousarray(M, dtype=np.float64)
    min_rank = min(int(min_rank), min(M.shape))
    V, tau, Tm, perm, r = cpqr_threshold(M, float(eps), min_rank)
    return dict(V=V, tau=tau, T=larft(V, tau), R=Tm[:r].copy(),
                resid=Tm[r:, r:].copy(), perm=perm, rank=int(r))


def check_pivots(R, context):
    """(`factor.py:57-68`, `kernels/__init__.py:211-223`)"""
    if R.shape[0] == 0:
        return
    d = np.abs(np.diag(R))
    if d[0] == 0.0:
        raise OracleSingularPivot(0, 0.0, context)
    bad = np.nonzero(d <= PIVOT_FLOOR * d[0])[0]
    if bad.size:
        raise OracleSingularPivot(int(bad[0]), R[bad[0], bad[0]], context)


def tri_solve_left(R, C):
    """R X = C, back substitution (`kernels/_numba.py:170-178`)."""
    X = np.array(C, dtype=np.float64, copy=True)
    k = R.shape[0]
    for i in range(k - 1, -1, -1):
        if i + 1 < k:
            X[i] -= R[i, i + 1:] @ X[i + 1:]
        X[i] /= R[i, i]
    return X


def tri_solve_right(R, C):
    """X R = C, forward over columns (`kernels/_numba.py:181-191`)."""
    Y = np.array(C, dtype=np.float64, copy=True)
    k = R.shape[0]
    for j in range(k):
        if j:
            Y[:, j] -= Y[:, :j] @ R[:j, j]
        Y[:, j] /= R[j, j]
    return Y


def spectral_norm(E):
    return 0.0 if E.size == 0 else float(np.linalg.svd(E, compute_uv=False)[0])


# ============================================================ transform records

class Panel:
    def __init__(self, V, tau, T):
        self.V, self.tau, self.T = V, tau, T

    @property
    def size(self):
        return self.V.size + self.tau.size + self.T.size


def _apply(panel, z, transpose):
    z2 = z.reshape(z.shape[0], -1)
    out = wy_apply(panel.V, panel.T, z2, transpose)
    return out.reshape(z.shape)


class RecElim:
    """Interior elimination (`factor.py:78-113`)."""
    kind = "elim"

    def __init__(self, rows, panel, cols_s, R_ss, cols_n, R_sn):
        self.rows, self.panel, self.cols_s, self.R_ss = rows, panel, cols_s, R_ss
        self.cols_n, self.R_sn = cols_n, R_sn

    payload = property(lambda s: s.panel.size + s.R_ss.size + s.R_sn.size)

    def qt(self, z):
        z[self.rows] = _apply(self.panel, z[self.rows], True)
        return z

    def w(self, x):
        xs = self.R_ss @ x[self.cols_s]
        if len(self.cols_n):
            xs += self.R_sn @ x[self.cols_n]
        x[self.cols_s] = xs
        return x

    def w_inv(self, y):
        rhs = y[self.cols_s]
        if len(self.cols_n):
            rhs = rhs - self.R_sn @ y[self.cols_n]
        y[self.cols_s] = tri_solve_left(self.R_ss, rhs.reshape(len(self.cols_s), -1)).reshape(rhs.shape)
        return y


class RecScale:
    """Interface scaling (`factor.py:116-142`)."""
    kind = "scale"

    def __init__(self, rows, panel, cols, R_pp):
        self.rows, self.panel, self.cols, self.R_pp = rows, panel, cols, R_pp

    payload = property(lambda s: s.panel.size + s.R_pp.size)

    def qt(self, z):
        z[self.rows] = _apply(self.panel, z[self.rows], True)
        return z

    def w(self, x):
        x[self.cols] = self.R_pp @ x[self.cols]
        return x

    def w_inv(self, y):
        v = y[self.cols]
        y[self.cols] = tri_solve_left(self.R_pp, v.reshape(len(self.cols), -1)).reshape(v.shape)
        return y


class RecSparsify:
    """Scaled sparsifier (`factor.py:145-205`, scaled flavour)."""
    kind = "sparsify"

    def __init__(self, rows, cols, panel, rank):
        self.rows, self.cols, self.panel, self.rank = rows, cols, panel, rank

    payload = property(lambda s: s.panel.size)
    q_panel = property(lambda s: s.panel)

    def qt(self, z):
        z[self.rows] = _apply(self.panel, z[self.rows], True)
        return z

    def w(self, x):
        x[self.cols] = _apply(self.panel, x[self.cols], True)
        return x

    def w_inv(self, y):
        y[self.cols] = _apply(self.panel, np.array(y[self.cols]), False)
        return y


class RecPerm:
    kind = "perm"

    def __init__(self, row_of_col):
        self.row_of_col = row_of_col

    payload = property(lambda s: 0)

    def qt(self, z):
        return z[self.row_of_col]


class RecDiag:
    kind = "diag"

    def __init__(self, scale):
        self.scale = scale

    payload = property(lambda s: s.scale.size)

    def w(self, x):
        return x * (self.scale[:, None] if x.ndim == 2 else self.scale)

    def w_inv(self, y):
        return y / (self.scale[:, None] if y.ndim == 2 else self.scale)


class OracleFactorization:
    def __init__(self, N, q_chain, w_chain, row_of_col, stats, ranks):
        self.N, self.q_chain, self.w_chain = N, q_chain, w_chain
        self.row_of_col, self.stats, self.ranks = row_of_col, stats, ranks

    @property
    def payload_scalars(self):
        seen, tot = set(), 0
        for r in self.q_chain + self.w_chain:
            if id(r) not in seen:
                seen.add(id(r))
                tot += r.payload
        return tot

    def apply_qt(self, b):
        z = np.array(b, dtype=np.float64, copy=True)
        for r in self.q_chain:
            z = r.qt(z)
        return z

    def apply_w(self, x):
        z = np.array(x, dtype=np.float64, copy=True)
        for r in self.w_chain:
            z = r.w(z)
        return z

    def solve_w(self, y):
        z = np.array(y, dtype=np.float64, copy=True)
        for r in reversed(self.w_chain):
            z = r.w_inv(z)
        return z


# ================================================================ block state

class BlockState:
    """Block-sparse trailing matrix (`factor.py:320-392`)."""

    def __init__(self, A, tree, equilibrate=True):
        n = int(A.ncols)
        indptr = np.asarray(A.indptr, np.int64)
        indices = np.asarray(A.indices, np.int64)
        data = np.asarray(A.data, np.float64)
        col_of = np.repeat(np.arange(n, dtype=np.int64), np.diff(indptr))
        self.scale = None
        if equilibrate:
            # sparse.py:142-166 — column 2-norms accumulated in entry order
            sq = np.zeros(n)
            np.add.at(sq, col_of, data ** 2)
            nrm = np.sqrt(sq)
            if (nrm == 0.0).any():
                raise OracleError(f"cannot equilibrate: column {int(np.nonzero(nrm == 0)[0][0])}")
            data = data / nrm[col_of]
            self.scale = nrm
        self.N = n
        self.tree = tree
        leaves = tree.leaf_clusters()
        self.rows_of = {c.id: np.asarray(c.rows if c.rows is not None else c.cols, np.int64).copy()
                        for c in leaves}
        self.cols_of = {c.id: np.asarray(c.cols, np.int64).copy() for c in leaves}
        self.rix = {c: set() for c in self.rows_of}      # row cluster -> col clusters
        self.cix = {c: set() for c in self.rows_of}      # col cluster -> row clusters
        self.blk = {}
        self.row_of_col = np.full(n, -1, np.int64)
        rown = np.empty(n, np.int64)
        coln = np.empty(n, np.int64)
        rpos = np.empty(n, np.int64)
        cpos = np.empty(n, np.int64)
        for c in leaves:
            rr, cc = self.rows_of[c.id], self.cols_of[c.id]
            rown[rr], coln[cc] = c.id, c.id
            rpos[rr], cpos[cc] = np.arange(len(rr)), np.arange(len(cc))
        # factor.py:352-374 — group entries by (row owner, col owner)
        ro, co = rown[indices], coln[col_of]
        key = ro * (len(tree.clusters) + 1) + co
        order = np.argsort(key, kind="stable")
        key_s = key[order]
        cut = np.r_[0, np.nonzero(np.diff(key_s))[0] + 1, len(key_s)]
        for a, b in zip(cut[:-1], cut[1:]):
            sel = order[a:b]
            i, j = int(ro[sel[0]]), int(co[sel[0]])
            B = np.zeros((len(self.rows_of[i]), len(self.cols_of[j])))
            np.add.at(B, (rpos[indices[sel]], cpos[col_of[sel]]), data[sel])
            self.put(i, j, B)

    def put(self, i, j, B):
        self.blk[(i, j)] = B
        self.rix[i].add(j)
        self.cix[j].add(i)

    def drop(self, i, j):
        self.blk.pop((i, j), None)
        self.rix[i].discard(j)
        self.cix[j].discard(i)

    def get(self, i, j):
        B = self.blk.get((i, j))
        return np.zeros((len(self.rows_of[i]), len(self.cols_of[j]))) if B is None else B

    def retire(self, s):
        for d in (self.rows_of, self.cols_of, self.rix, self.cix):
            d.pop(s, None)

    def total_cols(self):
        return sum(len(v) for v in self.cols_of.values())

    # ---------------------------------------------------------------- (a)
    def eliminate(self, s):
        """Interior elimination (`factor.py:402-493`)."""
        rows_s, cols_s = self.rows_of[s], self.cols_of[s]
        ns = len(cols_s)
        if ns == 0:
            self.retire(s)
            return None
        # panel rows: all of s, then nonzero rows of each coupled cluster (:416-431)
        plan = [(s, np.arange(len(rows_s)), True)]
        parts = [self.get(s, s)]
        for r in sorted(self.cix[s] - {s}):
            B = self.blk[(r, s)]
            ix = np.flatnonzero(B.any(axis=1))
            if len(ix):
                full = len(ix) == B.shape[0]
                plan.append((r, ix, full))
                parts.append(B if full else B[ix])
        heights = [len(ix) for _, ix, _ in plan]
        offs = np.r_[0, np.cumsum(heights)]
        stack_rows = np.concatenate([self.rows_of[r][ix] for r, ix, _ in plan])
        V, tau, R_ss = house_qr(np.vstack(parts))
        panel = Panel(V, tau, larft(V, tau))
        check_pivots(R_ss, f"pivot block of cluster {s}")
        # trailing columns: clusters touched by a panel row, kept if the
        # touched rows hold any nonzero (:436-463)
        row_clusters = [r for r, _, _ in plan]
        cand = sorted(set().union(*(self.rix[r] for r in row_clusters)) - {s})
        widths = [len(self.cols_of[c]) for c in cand]
        cw = np.r_[0, np.cumsum(widths)].astype(np.int64)
        buf = np.zeros((int(offs[-1]), int(cw[-1])))
        present = np.zeros(len(cand), bool)
        where = {c: q for q, c in enumerate(cand)}
        for (r, ix, full), o0, o1 in zip(plan, offs[:-1], offs[1:]):
            for c in self.rix[r]:
                q = where.get(c)
                if q is None:
                    continue
                sub = self.blk[(r, c)] if full else self.blk[(r, c)][ix]
                buf[o0:o1, cw[q]:cw[q + 1]] = sub
                present[q] = present[q] or bool(sub.any())
        cols_t = [c for q, c in enumerate(cand) if present[q]]
        if not present.all():
            keep = np.concatenate([np.full(widths[q], present[q]) for q in range(len(cand))]) \
                if cand else np.zeros(0, bool)
            buf = buf[:, keep]
        C = wy_apply(V, panel.T, buf, True)
        wo = np.r_[0, np.cumsum([len(self.cols_of[c]) for c in cols_t])].astype(np.int64)
        for c, w0, w1 in zip(cols_t, wo[:-1], wo[1:]):
            for (r, ix, full), o0, o1 in zip(plan, offs[:-1], offs[1:]):
                if r == s:
                    continue
                if full:
                    self.put(r, c, C[o0:o1, w0:w1].copy())
                else:
                    B = self.blk.get((r, c))
                    if B is None:
                        B = np.zeros((len(self.rows_of[r]), len(self.cols_of[c])))
                    B[ix] = C[o0:o1, w0:w1]
                    self.put(r, c, B)
        for r in list(self.cix[s]):
            self.drop(r, s)
        for c in list(self.rix[s]):
            self.drop(s, c)
        cols_n = (np.concatenate([self.cols_of[c] for c in cols_t]) if cols_t
                  else np.empty(0, np.int64))
        self.row_of_col[cols_s] = rows_s
        rec = RecElim(stack_rows, panel, cols_s.copy(), R_ss, cols_n, C[:ns].copy())
        rec.cid = s
        self.retire(s)
        return rec

    # ---------------------------------------------------------------- (b)
    def scale_iface(self, p):
        """Rescale interface p's diagonal block to I (`factor.py:504-532`)."""
        npp = len(self.cols_of[p])
        if npp == 0:
            return None
        V, tau, R_pp = house_qr(self.get(p, p))
        panel = Panel(V, tau, larft(V, tau))
        check_pivots(R_pp, f"diagonal block of interface {p}")
        for c in sorted(self.rix[p] - {p}):
            self.blk[(p, c)] = wy_apply(V, panel.T, self.blk[(p, c)], True)
        for r in sorted(self.cix[p] - {p}):
            self.blk[(r, p)] = tri_solve_right(R_pp, self.blk[(r, p)])
        self.put(p, p, np.eye(npp))
        rec = RecScale(self.rows_of[p].copy(), panel, self.cols_of[p].copy(), R_pp)
        rec.cid = p
        return rec

    # ---------------------------------------------------------------- (c)
    def sparsify_iface(self, p, eps):
        """Scaled-mode compression of interface p (`factor.py:536-658`)."""
        cols_p, rows_p = self.cols_of[p], self.rows_of[p]
        npp = len(cols_p)
        if npp == 0:
            return None, 0.0, None
        us = sorted(self.cix[p] - {p})
        cs = sorted(self.rix[p] - {p})
        Anp = np.vstack([self.blk[(u, p)] for u in us]) if us else np.zeros((0, npp))
        Apn = np.hstack([self.blk[(p, c)] for c in cs]) if cs else np.zeros((npp, 0))
        M = np.hstack([Anp.T, Apn])
        cn = np.sqrt(np.einsum("ij,ij->j", M, M)) if M.size else np.zeros(M.shape[1])
        maxcol = float(cn.max()) if M.size else 0.0
        ratio = 0.0 if maxcol == 0.0 else min(eps / maxcol, 0.999999)
        Mk = M
        if maxcol > 0.0 and M.shape[1] > 4 * M.shape[0]:
            keep = cn >= ratio * maxcol
            if not keep.all():
                Mk = np.ascontiguousarray(M[:, keep])
        res = rrqr_threshold(Mk, ratio)
        r = res["rank"]
        info = dict(rank=r, ratio=ratio, maxcol=maxcol, ncols=M.shape[1], kept=Mk.shape[1])
        if r >= npp:
            return None, 0.0, info
        panel = Panel(res["V"], res["tau"], res["T"])
        QtM = wy_apply(panel.V, panel.T, M, True)
        nu = Anp.shape[0]
        E1, E2 = QtM[r:, :nu].T, QtM[r:, nu:]
        off = 0
        for u in us:
            h = len(self.rows_of[u])
            blk = QtM[:r, off:off + h].T
            off += h
            if blk.size:
                self.put(u, p, blk.copy())
            else:
                self.drop(u, p)
        for c in cs:
            w = len(self.cols_of[c])
            blk = QtM[:r, off:off + w]
            off += w
            if blk.size:
                self.put(p, c, blk.copy())
            else:
                self.drop(p, c)
        dropped = max(spectral_norm(E1), spectral_norm(E2))
        rec = RecSparsify(rows_p.copy(), cols_p.copy(), panel, r)
        rec.cid = p
        self.row_of_col[cols_p[r:]] = rows_p[r:]
        self.rows_of[p] = rows_p[:r].copy()
        self.cols_of[p] = cols_p[:r].copy()
        if r:
            self.put(p, p, np.eye(r))
        else:
            self.drop(p, p)
            for u in us:
                self.drop(u, p)
            for c in cs:
                self.drop(p, c)
        return rec, dropped, info

    # ---------------------------------------------------------------- (d)
    def merge(self, lev):
        """Fragments -> depth lev-1 parents (`factor.py:713-748`)."""
        parent, ro, co = {}, {}, {}
        rows, cols = {}, {}
        for P in self.tree.active_at(lev - 1):
            a = b = 0
            for k in P.children:
                parent[k], ro[k], co[k] = P.id, a, b
                a += len(self.rows_of[k])
                b += len(self.cols_of[k])
            rows[P.id] = (np.concatenate([self.rows_of[k] for k in P.children])
                          if P.children else np.empty(0, np.int64))
            cols[P.id] = (np.concatenate([self.cols_of[k] for k in P.children])
                          if P.children else np.empty(0, np.int64))
        old = self.blk
        self.rows_of, self.cols_of = rows, cols
        self.rix = {c: set() for c in rows}
        self.cix = {c: set() for c in rows}
        self.blk = {}
        for (i, j), B in old.items():
            if B.size == 0:
                continue
            Pi, Pj = parent[i], parent[j]
            tgt = self.blk.get((Pi, Pj))
            if tgt is None:
                tgt = np.zeros((len(rows[Pi]), len(cols[Pj])))
                self.put(Pi, Pj, tgt)
            tgt[ro[i]:ro[i] + B.shape[0], co[j]:co[j] + B.shape[1]] = B


def factorize(A, tree, eps=1e-3, *, sparsify=True, scaling=True, skip=2,
              sparsify_min=40, equilibrate=True, stop_level=None):
    """Level driver (`factor.py:771-911`), scaled mode, scale_every=1.
    ``stop_level`` (diagnostics): return the ranks/stats logged down to that
    level without finishing the factorization."""
    st = BlockState(A, tree, equilibrate)
    L = tree.L
    q_chain = []
    w_chain = [RecDiag(st.scale)] if equilibrate else []
    stats, ranks = [], []
    fac = {l: sorted(c.id for c in tree.factor_at(l)) for l in range(1, L + 1)}
    pend = {l: sorted(c.id for c in tree.sparsify_at(l)) for l in range(1, L + 1)}
    for lev in range(L, 0, -1):
        row = dict(level=lev, cols_before=st.total_cols(), n_factored=0, factored_cols=0,
                   n_scaled=0, n_sparsified=0, fine_retired=0, dropped_max=0.0)
        for s in fac[lev]:
            row["factored_cols"] += len(st.cols_of[s])
            rec = st.eliminate(s)
            row["n_factored"] += 1
            if rec is not None:
                q_chain.append(rec)
                w_chain.append(rec)
        if sparsify and (L - lev + 1) > skip and lev >= 2 and pend[lev]:
            todo = [p for p in pend[lev] if len(st.cols_of[p]) >= sparsify_min]
            if scaling:
                for p in todo:
                    rec = st.scale_iface(p)
                    if rec is not None:
                        q_chain.append(rec)
                        w_chain.append(rec)
                        row["n_scaled"] += 1
            for p in todo:
                before = len(st.cols_of[p])
                rec, dropped, info = st.sparsify_iface(p, eps) if scaling else (None, 0.0, None)
                if info is not None:
                    ranks.append((lev, p, info["rank"], before))
                if rec is not None:
                    q_chain.append(rec)
                    w_chain.append(rec)
                    row["n_sparsified"] += 1
                    row["fine_retired"] += before - len(st.cols_of[p])
                    row["dropped_max"] = max(row["dropped_max"], dropped)
        sizes = [len(st.cols_of[p]) for p in pend[lev]]
        if sizes:
            q = np.percentile(sizes, [25, 50, 75])
            row.update(iface_q1=float(q[0]), iface_q2=float(q[1]), iface_q3=float(q[2]),
                       iface_max=int(max(sizes)))
        else:
            row.update(iface_q1=0.0, iface_q2=0.0, iface_q3=0.0, iface_max=0)
        row["cols_after"] = st.total_cols()
        row["trailing_nnz"] = int(sum(np.count_nonzero(B) for B in st.blk.values()))
        row["trailing_blocks"] = len(st.blk)
        if lev >= 2:
            st.merge(lev)
        stats.append(row)
        if stop_level is not None and lev <= stop_level:
            return OracleFactorization(st.N, q_chain, w_chain, st.row_of_col, stats, ranks)
    if (st.row_of_col < 0).any():
        raise OracleError("columns never factored")
    q_chain.append(RecPerm(st.row_of_col))
    return OracleFactorization(st.N, q_chain, w_chain, st.row_of_col, stats, ranks)
