"""CPU ORACLE — test infrastructure only, never the product path.

Plain numpy/scipy restatement of the reference FIND selected-inversion path
(arXiv 1104.0623; reference package ``find_selinv`` 0.1.0 under
/root/reference/pkg/src/find_selinv).  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference`` arm) may
import this module, and only as the checker / CPU baseline.

Parity pin: this restatement is checked against golden vectors produced by the
reference itself (``tests/golden/make_golden.py`` imports ``find_selinv`` read-only
in the build container and writes ``tests/golden/*.npz``); see
``tests/test_oracle_golden.py``.

Every function cites the reference file:line it restates.  Line numbers refer to
/root/reference/pkg/src/find_selinv/<module>.py.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np
import scipy.linalg as la
import scipy.sparse as sp


class OracleSingularPivot(Exception):
    """Mirrors errors.SingularPivotError (errors.py:8-18)."""

    def __init__(self, message, node=None, cluster=None):
        super().__init__(message)
        self.node = node
        self.cluster = cluster


# ---------------------------------------------------------------------------
# Tree and node sets (mesh.py:176-290)
# ---------------------------------------------------------------------------


@dataclass(eq=False)
class OCluster:
    label: int
    x0: int
    y0: int
    w: int
    h: int
    level: int
    children: tuple = ()
    parent: "OCluster | None" = None
    nodes: np.ndarray = None
    boundary: np.ndarray = None
    private_inner: np.ndarray = None

    @property
    def is_leaf(self):
        return not self.children


def rect_nodes(nx, x0, y0, w, h):
    """mesh.py:170-173 — ascending ids of a rectangle (id = x + nx*y)."""
    ys = np.arange(y0, y0 + h, dtype=np.int64) * nx
    xs = np.arange(x0, x0 + w, dtype=np.int64)
    return (ys[:, None] + xs[None, :]).ravel()


def build_tree(nx, ny, leaf_max):
    """mesh.py:176-206 — recursive bisection of the longer side (ties -> x),
    ceil half first, heap labels 1 / 2g / 2g+1, leaf when both sides <= leaf_max."""
    if leaf_max < 1:
        raise ValueError("leaf_max must be >= 1")
    by_label = {}

    def make(label, x0, y0, w, h, level, parent):
        c = OCluster(label, x0, y0, w, h, level, parent=parent,
                     nodes=rect_nodes(nx, x0, y0, w, h))
        by_label[label] = c
        if w <= leaf_max and h <= leaf_max:
            return c
        if w >= h:
            wl = (w + 1) // 2
            c.children = (make(2 * label, x0, y0, wl, h, level + 1, c),
                          make(2 * label + 1, x0 + wl, y0, w - wl, h, level + 1, c))
        else:
            hl = (h + 1) // 2
            c.children = (make(2 * label, x0, y0, w, hl, level + 1, c),
                          make(2 * label + 1, x0, y0 + hl, w, h - hl, level + 1, c))
        return c

    root = make(1, 0, 0, nx, ny, 0, None)
    return root, by_label


def _adjacency(matrix: sp.csr_matrix) -> sp.csr_matrix:
    """operators.py:84-93 — off-diagonal stored pattern (explicit zeros kept)."""
    c = matrix.tocoo()
    off = c.row != c.col
    return sp.csr_matrix((np.ones(int(off.sum()), dtype=np.int8), (c.row[off], c.col[off])),
                         shape=c.shape)


def _in_rect(nodes, nx, c):
    x = nodes % nx
    y = nodes // nx
    return (x >= c.x0) & (x < c.x0 + c.w) & (y >= c.y0) & (y < c.y0 + c.h)


def boundary_nodes(adj: sp.csr_matrix, nx, c):
    """mesh.py:209-221 — nodes of C with at least one neighbour outside C.
    Restated with a rectangle test instead of a full sparse mat-vec."""
    nodes = c.nodes
    sub = adj[nodes]
    outside = ~_in_rect(sub.indices.astype(np.int64), nx, c)
    counts = np.add.reduceat(outside.astype(np.int64), sub.indptr[:-1]) if sub.nnz else np.zeros(nodes.size, np.int64)
    # reduceat on empty rows returns the next value; mask rows with no entries
    empty = np.diff(sub.indptr) == 0
    counts[empty] = 0
    return nodes[counts > 0]


def adjacent_nodes(adj: sp.csr_matrix, nx, c):
    """mesh.py:224-232 — nodes outside C adjacent to C (the complement boundary)."""
    sub = adj[c.nodes]
    cols = sub.indices.astype(np.int64)
    cols = cols[~_in_rect(cols, nx, c)]
    return np.unique(cols)


def annotate(by_label, adj, nx):
    """mesh.py:255-264 + mesh.py:235-252 — B, and S = (B_l U B_r) \\ B_parent
    (leaves: S = C \\ B)."""
    for c in sorted(by_label.values(), key=lambda c: (-c.level, c.label)):
        c.boundary = boundary_nodes(adj, nx, c)
        if c.is_leaf:
            c.private_inner = np.setdiff1d(c.nodes, c.boundary, assume_unique=True)
        else:
            l, r = c.children
            union = np.union1d(l.boundary, r.boundary)
            c.private_inner = np.setdiff1d(union, c.boundary, assume_unique=True)


def complement_sets(root, by_label, adj, nx):
    """mesh.py:267-290 — complement boundary B_{-c} = adjacent(C) and
    S_{-c} = (B_{-parent} U B_sibling) \\ B_{-c}; empty for the root."""
    empty = np.array([], dtype=np.int64)
    out = {-1: (empty, empty)}
    stack = [root]
    while stack:
        c = stack.pop()
        if c.parent is not None:
            b = adjacent_nodes(adj, nx, c)
            a, bb = c.parent.children
            sib = bb if a is c else a
            merged = np.union1d(out[-c.parent.label][0], sib.boundary)
            s = np.setdiff1d(merged, b, assume_unique=True)
            out[-c.label] = (b, s)
        stack.extend(reversed(c.children))
    return out


# ---------------------------------------------------------------------------
# Ledger (kernels.py:48-146, naive variants only)
# ---------------------------------------------------------------------------


@dataclass
class OLedger:
    multiplications: Fraction = Fraction(0)
    by_kernel: dict = field(default_factory=dict)

    def add(self, kernel, count):
        count = Fraction(count)
        self.multiplications += count
        self.by_kernel[kernel] = self.by_kernel.get(kernel, Fraction(0)) + count


def naive_dense_count(s, b):
    """kernels.py:90 — s^3/3 + s^2 b + s b^2."""
    s, b = Fraction(s), Fraction(b)
    return s ** 3 / 3 + s * s * b + s * b * b


def sigma_naive_count(s, b):
    """kernels.py:91 — s^2 b + 3 s b^2."""
    s, b = Fraction(s), Fraction(b)
    return s * s * b + 3 * s * b * b


# ---------------------------------------------------------------------------
# Dense kernels (kernels.py:237-266, 363-392)
# ---------------------------------------------------------------------------


def lu_checked(a, labels, rtol):
    """kernels.py:237-252 — LU with partial pivoting + relative singular-pivot test."""
    if a.shape[0] == 0:
        return None
    scale = float(np.abs(a).max()) if a.size else 0.0
    if scale == 0.0:
        raise OracleSingularPivot("zero pivot block", node=int(labels[0]))
    lu, piv = la.lu_factor(a, check_finite=False)
    diag = np.abs(np.diagonal(lu))
    bad = np.nonzero(diag < rtol * scale)[0]
    if bad.size:
        raise OracleSingularPivot(f"singular pivot at elimination position {bad[0]}",
                                  node=int(labels[min(int(bad[0]), len(labels) - 1)]))
    return lu, piv


def schur_update(ass, asb, abs_, abb, s_labels, ledger, rtol=1e-12):
    """kernels.py:363-380 — U = Abb - L Asb, L = Abs Ass^{-1} (zgetrf + zgetrs trans)."""
    s, b = ass.shape[0], abb.shape[0]
    if s == 0:
        return abb.astype(np.complex128, copy=True), np.zeros((b, 0), np.complex128)
    lu = lu_checked(ass, s_labels, rtol)
    if b:
        l_fac = la.lu_solve(lu, abs_.T, trans=1, check_finite=False).T
    else:
        l_fac = np.zeros((0, s), np.complex128)
    u = abb - l_fac @ asb
    ledger.add("naive_dense", naive_dense_count(s, b))
    return u, l_fac


def sigma_update(sss, ssb, sbs, sbb, l_fac, ledger):
    """kernels.py:383-392 — R = Sbb - L Ssb - Sbs L^H + (L Sss) L^H."""
    s = sss.shape[0]
    b = sbb.shape[0]
    if s == 0:
        return sbb.astype(np.complex128, copy=True)
    lh = l_fac.conj().T
    r = sbb - l_fac @ ssb - sbs @ lh + (l_fac @ sss) @ lh
    ledger.add("sigma_naive", sigma_naive_count(s, b))
    return r


# ---------------------------------------------------------------------------
# Passes (solver.py:97-132, 188-243, 256-375, 392-418, 586-701)
# ---------------------------------------------------------------------------


def extract(m: sp.csr_matrix, rows, cols):
    """operators.py:202-219 — dense gather of a sparse block by label lists."""
    rows = np.asarray(rows, np.int64)
    cols = np.asarray(cols, np.int64)
    if rows.size == 0 or cols.size == 0:
        return np.zeros((rows.size, cols.size), np.complex128)
    return m[rows][:, cols].toarray().astype(np.complex128)


def merge_matrix(m, left, right, u_left, u_right):
    """solver.py:97-108 — [[U_l, M(l,r)], [M(r,l), U_r]]."""
    p, q = left.size, right.size
    out = np.zeros((p + q, p + q), np.complex128)
    if p:
        out[:p, :p] = u_left
    if q:
        out[p:, p:] = u_right
    if p and q:
        out[:p, p:] = extract(m, left, right)
        out[p:, :p] = extract(m, right, left)
    return out


def merge_permutation(left, right, s_set):
    """solver.py:111-132 — reorder to [S_l, S_r, B_l, B_r]."""
    labels = np.concatenate([left, right])
    in_sl = np.isin(left, s_set)
    in_sr = np.isin(right, s_set)
    pl = np.arange(left.size)
    pr = left.size + np.arange(right.size)
    perm = np.concatenate([pl[in_sl], pr[in_sr], pl[~in_sl], pr[~in_sr]])
    s_count = int(in_sl.sum() + in_sr.sum())
    return perm, labels[perm], s_count


@dataclass
class OracleResult:
    gr_diag: np.ndarray
    gless_diag: np.ndarray | None
    ledger: OLedger
    timings: dict
    offdiag: dict | None = None        # G^r on adjacent pairs (solver.py:454-484, 666-669)
    offdiag_gless: dict | None = None  # G^< on the same pairs (_extended_extraction, solver.py:487-507)


class FindOracle:
    """Energy-independent plan (tree + sets) built once; ``solve`` per energy.

    Mirrors reference ``solve`` (solver.py:586-701) with kernel='naive',
    tiling='full-leaves'."""

    def __init__(self, nx, ny, pattern: sp.csr_matrix, leaf_max=2):
        self.nx, self.ny = nx, ny
        self.n = nx * ny
        self.leaf_max = leaf_max
        self.root, self.by_label = build_tree(nx, ny, leaf_max)
        adj = _adjacency(pattern.tocsr())
        annotate(self.by_label, adj, nx)
        self.comps = complement_sets(self.root, self.by_label, adj, nx)
        self.bottom_up = sorted(self.by_label.values(), key=lambda c: (-c.level, c.label))
        self._off = self._offl = self._adj = None  # off-diagonal harvest state (solve(compute_offdiag=True))

    # solver.py:188-232
    def _eliminate(self, a, sg, left, right, ul, ur, rl, rr, s_set, label, want_sigma, ledger, rtol):
        amat = merge_matrix(a, left, right, ul, ur)
        perm, labels, sc = merge_permutation(left, right, s_set)
        amat = amat[np.ix_(perm, perm)]
        try:
            u, l_fac = schur_update(amat[:sc, :sc], amat[:sc, sc:], amat[sc:, :sc], amat[sc:, sc:],
                                    labels[:sc], ledger, rtol)
        except OracleSingularPivot as exc:
            exc.cluster = label
            raise
        rmat = None
        if want_sigma:
            smat = merge_matrix(sg, left, right, rl, rr)[np.ix_(perm, perm)]
            rmat = sigma_update(smat[:sc, :sc], smat[:sc, sc:], smat[sc:, :sc], smat[sc:, sc:],
                                l_fac, ledger)
        # solver.py:234-243 — store sorted by B label
        b_labels = labels[sc:]
        order = np.argsort(b_labels, kind="stable")
        u = u[np.ix_(order, order)]
        if rmat is not None:
            rmat = rmat[np.ix_(order, order)]
        return u, rmat

    def solve(self, a: sp.csr_matrix, sigma: sp.csr_matrix | None, compute_gless=True, pivot_rtol=1e-12,
              compute_offdiag=False):
        import time

        t0 = time.perf_counter()
        a = a.tocsr()
        sg = sigma.tocsr() if sigma is not None else None
        ledger = OLedger()
        empty = np.array([], np.int64)
        z = np.zeros((0, 0), np.complex128)
        pos = {}
        # upward_pass, solver.py:256-308
        for c in self.bottom_up:
            if c.parent is None:
                continue
            if c.is_leaf:
                order = np.concatenate([c.private_inner, c.boundary])
                seed = extract(a, order, order)
                rseed = extract(sg, order, order) if compute_gless else None
                pos[c.label] = self._eliminate(a, sg, order, empty, seed, z, rseed, z, c.private_inner,
                                               c.label, compute_gless, ledger, pivot_rtol)
            else:
                i, j = c.children
                pos[c.label] = self._eliminate(a, sg, i.boundary, j.boundary, pos[i.label][0], pos[j.label][0],
                                               pos[i.label][1], pos[j.label][1], c.private_inner,
                                               c.label, compute_gless, ledger, pivot_rtol)
        t1 = time.perf_counter()
        gr = np.zeros(self.n, np.complex128)
        gl = np.zeros(self.n, np.complex128) if compute_gless else None
        filled = np.zeros(self.n, bool)
        self._off = {} if compute_offdiag else None
        self._offl = {} if (compute_offdiag and compute_gless) else None
        self._adj = _adjacency(a) if compute_offdiag else None
        # downward_pass, solver.py:311-375 (DFS, negative data freed per subtree)
        neg = {-1: (z, z if compute_gless else None)}
        stack = [(self.root, False)]
        while stack:
            c, done = stack.pop()
            if done:
                if c.parent is not None:
                    del neg[-c.label]
                continue
            if c.parent is not None:
                p = c.parent
                a0, a1 = p.children
                sib = a1 if a0 is c else a0
                left = self.comps[-p.label][0]
                b_set, s_set = self.comps[-c.label]
                pu, pr = neg[-p.label]
                su, sr = pos[sib.label]
                neg[-c.label] = self._eliminate(a, sg, left, sib.boundary, pu, su, pr, sr, s_set,
                                                -c.label, compute_gless, ledger, pivot_rtol)
            if c.is_leaf:
                self._leaf(c, a, sg, neg[-c.label], gr, gl, filled, ledger, compute_gless, pivot_rtol)
                if c.parent is not None:
                    del neg[-c.label]
            else:
                stack.append((c, True))
                for ch in reversed(c.children):
                    stack.append((ch, False))
        t2 = time.perf_counter()
        if not filled.all():
            raise RuntimeError("extraction did not cover every node")
        return OracleResult(gr, gl, ledger, {"upward": t1 - t0, "downward_extract": t2 - t1, "total": t2 - t0},
                            self._off, self._offl)

    def _leaf(self, leaf, a, sg, negdata, gr, gl, filled, ledger, compute_gless, rtol):
        """solver.py:392-418 (_final_elimination), 383-389 (_invert), 660-669 (sandwich, harvest)."""
        ring = self.comps[-leaf.label][0]
        nodes = leaf.nodes
        nu, nr = negdata
        try:
            u_f, l_fac = schur_update(nu, extract(a, ring, nodes), extract(a, nodes, ring),
                                      extract(a, nodes, nodes), ring, ledger, rtol)
        except OracleSingularPivot as exc:
            exc.cluster = leaf.label
            raise
        try:
            g = np.linalg.inv(u_f) if u_f.size else u_f.copy()
        except np.linalg.LinAlgError as exc:
            raise OracleSingularPivot(f"singular final block: {exc}", cluster=leaf.label) from exc
        ledger.add("dense_inverse", Fraction(u_f.shape[0]) ** 3)
        new = ~filled[nodes]
        gr[nodes[new]] = np.diagonal(g)[new]
        if compute_gless:
            r_f = sigma_update(nr, extract(sg, ring, nodes), extract(sg, nodes, ring),
                               extract(sg, nodes, nodes), l_fac, ledger)
            gless = (g @ r_f) @ g.conj().T
            ledger.add("gless_sandwich", 2 * Fraction(g.shape[0]) ** 3)
            gl[nodes[new]] = np.diagonal(gless)[new]
        filled[nodes] = True
        if self._off is not None:
            self._leaf_offdiag(leaf, a, sg, ring, nodes, nu, nr, g, ledger)

    def _leaf_offdiag(self, leaf, a, sg, ring, nodes, nu, nr, g, ledger):
        """leaf_extract_offdiag (solver.py:454-484), first writer wins (solver.py:666-669):
        pairs inside the leaf from G(C,C); cross pairs by one back-substitution each way.
        G^< on the same pairs from the ring+leaf system as _extended_extraction does
        (solver.py:487-507): g_t = M^-1, G^<_t = g_t S_t g_t^H."""
        adj = self._adj
        labels = np.concatenate([ring, nodes])
        t = ring.size
        gl_t = None
        if self._offl is not None:
            m = merge_matrix(a, ring, nodes, nu, extract(a, nodes, nodes))
            s_t = merge_matrix(sg, ring, nodes, nr, extract(sg, nodes, nodes))
            g_t = np.linalg.inv(m)
            gl_t = (g_t @ s_t) @ g_t.conj().T

        def put(i, j, gval, li, lj):
            key = (int(labels[li]), int(labels[lj]))
            if key not in self._off:
                self._off[key] = complex(gval)
                if gl_t is not None:
                    self._offl[key] = complex(gl_t[li, lj])

        sub = adj[nodes][:, nodes].tocoo()
        for i, j in zip(sub.row, sub.col):
            put(i, j, g[i, j], t + i, t + j)
        if t:
            a_bc = extract(a, ring, nodes)
            a_cb = extract(a, nodes, ring)
            g_bc = -np.linalg.solve(nu, a_bc @ g)
            g_cb = -np.linalg.solve(nu.conj().T, (g @ a_cb).conj().T).conj().T
            ledger.add("offdiag_backsub", 2 * (Fraction(t) ** 2 * nodes.size + t * Fraction(nodes.size) ** 2))
            cross = adj[ring][:, nodes].tocoo()
            for i, j in zip(cross.row, cross.col):
                put(i, j, g_bc[i, j], i, t + j)
                put(j, i, g_cb[j, i], t + j, i)


def dense_gr_diag(a):
    """oracle.py:22-31."""
    return np.ascontiguousarray(np.diagonal(np.linalg.inv(np.asarray(a, np.complex128))))


def dense_gless_diag(a, sigma):
    """oracle.py:34-46 — diag(A^{-1} S A^{-H}) by two dense solves."""
    a = np.asarray(a, np.complex128)
    x = np.linalg.solve(a, np.asarray(sigma, np.complex128))
    g = np.linalg.solve(a, x.conj().T).conj().T
    return np.ascontiguousarray(np.diagonal(g))


def work_naive(oracle: FindOracle, compute_gless=True) -> Fraction:
    """Exact reference ledger (kernel='naive') from set sizes alone:
    kernels.py:379,391 per elimination, solver.py:388,664 per leaf."""
    w = Fraction(0)
    for c in oracle.by_label.values():
        if c.parent is None:
            continue
        s, b = c.private_inner.size, c.boundary.size
        if s:
            w += naive_dense_count(s, b) + (sigma_naive_count(s, b) if compute_gless else 0)
        bn, sn = oracle.comps[-c.label]
        s, b = sn.size, bn.size
        if s:
            w += naive_dense_count(s, b) + (sigma_naive_count(s, b) if compute_gless else 0)
        if c.is_leaf:
            t, cc = bn.size, c.nodes.size
            if t:
                w += naive_dense_count(t, cc) + (sigma_naive_count(t, cc) if compute_gless else 0)
            w += Fraction(cc) ** 3 + (2 * Fraction(cc) ** 3 if compute_gless else 0)
    if oracle.root.is_leaf:
        cc = oracle.root.nodes.size
        w += Fraction(cc) ** 3 + (2 * Fraction(cc) ** 3 if compute_gless else 0)
    return w
