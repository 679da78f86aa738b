"""Pass-level drop-in API: ``upward_pass``, ``downward_pass`` and the leaf extractions
(mirrors find_selinv/solver.py:256-375 and 421-484), on the B200 path.

``solve`` runs both passes and the extraction as one level-batched device schedule; these
functions expose the same stages one at a time with the reference's signatures and return
values (``ClusterData`` per cluster label, ``DenseBlock`` per leaf), for callers that inspect or
reuse the intermediate blocks.  The arithmetic runs on the device:

* upward_pass / downward_pass run the plan's launch groups of that pass (find_solve_groups)
  and copy the stored U / R blocks of every elimination out of the block arenas
  (find_plan_elim_out), sorted by boundary label as the reference stores them
  (solver.py:234-243).  downward_pass first writes the caller's upward blocks into the
  upward arena, so it consumes exactly the ``cluster_data`` it is given.
* the leaf extractions run one elimination through the device shim (find_schur_sigma_update,
  the same kernels as the batched path): the final Schur step (solver.py:392-418), the leaf
  inverse as the elimination of [[U_f, I], [I, 0]] (U = -U_f^{-1}), and the back-substitutions
  of leaf_extract_offdiag as L = A(B,S) A(S,S)^{-1} outputs; the small G R_f G^H sandwich and
  coupling products use torch matmul on the device.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import NativeLibraryError, SingularPivotError, TreeStateError
from .ledger import FlopLedger, flop_model
from .operators import DenseBlock, SparseOperator

__all__ = ["ClusterData", "upward_pass", "downward_pass", "leaf_extract_gr", "leaf_extract_gless",
           "leaf_extract_offdiag"]


@dataclass
class ClusterData:
    """solver.py:74-79: updated operator and scattering blocks over one cluster's boundary."""

    u: DenseBlock
    r: DenseBlock | None = None


# ------------------------------------------------------------------------------ helpers
_TINY = float(np.finfo(np.float64).tiny)  # pivot floor of the inverse / back-substitution eliminations: exact zeros only

def _dev():
    import torch

    if not torch.cuda.is_available():
        raise NativeLibraryError("the FIND B200 path needs a CUDA device (there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _extract(op: SparseOperator, rows, cols) -> np.ndarray:
    rows = np.asarray(rows, np.int64)
    cols = np.asarray(cols, np.int64)
    if rows.size == 0 or cols.size == 0:
        return np.zeros((rows.size, cols.size), np.complex128)
    return op.matrix[rows][:, cols].toarray().astype(np.complex128)


def _device_elimination(ass, asb, abs_, abb, sig=None, rtol=1e-12, want_l=False):
    """One elimination on the device (find_schur_sigma_update): U, R (or None), L (or None) as
    torch device tensors; raises SingularPivotError(node=position) on a failing pivot."""
    import torch

    dev = _dev()
    s, b = ass.shape[0], abb.shape[0]
    t = lambda x: x.to(dev).contiguous() if isinstance(x, torch.Tensor) else \
        torch.from_numpy(np.ascontiguousarray(x, dtype=np.complex128)).to(dev)
    ins = [t(x) for x in (ass, asb, abs_, abb)]
    sg = [t(x) for x in sig] if sig is not None else [None] * 4
    u = torch.zeros((b, b), dtype=torch.complex128, device=dev)
    r = torch.zeros((b, b), dtype=torch.complex128, device=dev) if sig is not None else None
    lo = torch.zeros((b, s), dtype=torch.complex128, device=dev) if want_l else None
    st = _native.FindStatus()
    ptr = lambda x: C.c_void_p(x.data_ptr()) if x is not None and x.numel() else C.c_void_p(0)
    rc = _native.lib().find_schur_sigma_update(
        s, b, *[ptr(x) for x in ins], *[ptr(x) for x in sg], float(rtol), ptr(u), ptr(r), ptr(lo), -1,
        C.c_void_p(torch.cuda.current_stream(dev).cuda_stream), C.byref(st))
    if rc == _native.FIND_ESINGULAR:
        raise SingularPivotError(st.text, node=int(st.node_id) if st.node_id >= 0 else None)
    if rc != _native.FIND_OK:
        if rc == _native.FIND_EINVAL:
            raise ValueError(st.text)
        raise NativeLibraryError(f"find_schur_sigma_update failed ({rc}): {st.text}")
    return u, r, lo


def _device_inverse(m, label):
    """m^{-1} as minus the Schur complement of [[m, I], [I, 0]] (solver.py:383-389 semantics)."""
    import torch

    c = m.shape[0]
    if c == 0:
        return torch.zeros((0, 0), dtype=torch.complex128, device=_dev())
    eye = np.eye(c, dtype=np.complex128)
    try:
        u, _, _ = _device_elimination(m, eye, eye, np.zeros((c, c), np.complex128), rtol=_TINY)
    except SingularPivotError as exc:
        raise SingularPivotError(f"singular final block: {exc}", cluster=label) from exc
    return -u


def _plan_for_tree(tree, a: SparseOperator):
    from .plan import plan_for
    from .solver import _csr_sorted

    am = _csr_sorted(a.matrix)
    if a.n != tree.mesh.n:
        raise ValueError(f"operator size {a.n} does not match mesh with {tree.mesh.n} nodes")
    plan, _ = plan_for(tree.mesh.nx, tree.mesh.ny, am.indptr, am.indices, tree.leaf_max)
    return plan, am


def _elim_layout(plan):
    lay = plan.cache.get("elim_layout")
    if lay is None:
        L = _native.lib()
        ne = plan.info["n_elims"]
        oa = np.zeros(ne, np.int32)
        oo = np.zeros(ne, np.int64)
        L.find_plan_elim_out(plan.handle, oa.ctypes.data_as(C.POINTER(C.c_int32)), oo.ctypes.data_as(C.POINTER(C.c_int64)))
        ae = np.zeros(4, np.int64)
        L.find_plan_arena_elems(plan.handle, ae.ctypes.data_as(C.POINTER(C.c_int64)))
        lay = (oa, oo, ae)
        plan.cache["elim_layout"] = lay
    return lay


def _arena_views(plan, ws, n_energies=1):
    """Torch complex views of the four block arenas inside the workspace (energy 0 slices)."""
    import torch

    _, _, ae = _elim_layout(plan)
    views, base = [], 256
    for k in range(4):
        nb = int(ae[k]) * 16
        views.append(ws[base:base + nb].view(torch.complex128))
        base += n_energies * nb
    return views


def _values(plan, am, sigma, compute_gless):
    from .solver import _sigma_prepare

    a_vals = np.ascontiguousarray(am.data, np.complex128)[None, :]
    s_vals, ssym, herm = None, 0, False
    if compute_gless:
        if sigma is None:
            raise ValueError("compute_gless requires a scattering matrix")
        s_vals, ssym, herm = _sigma_prepare(plan, am, sigma)
    return a_vals, s_vals, ssym, herm


def _charge(ledger, plan, mask, config, sigma_herm):
    from .ledger import plan_ledger

    if ledger is None or not mask.any():
        return
    led = plan_ledger(plan.kind[mask], plan.s[mask], plan.b[mask], config.kernel, config.compute_gless, sigma_herm,
                      config.sigma_mode)
    for k, v in led.by_kernel.items():
        ledger.add(k, v)


# ------------------------------------------------------------------------------ passes
def upward_pass(tree, a: SparseOperator, sigma: SparseOperator | None, config, ledger: FlopLedger | None = None,
                engine=None) -> dict[int, ClusterData]:
    """solver.py:256-308: eliminate private inner nodes leaves-to-root; data for every non-root
    cluster (U and, with compute_gless, R over its boundary, ascending labels)."""
    import torch

    plan, am = _plan_for_tree(tree, a)
    dev = _dev()
    a_vals, s_vals, ssym, herm = _values(plan, am, sigma, config.compute_gless)
    a_d = torch.from_numpy(a_vals).to(dev)
    s_d = torch.from_numpy(s_vals).to(dev) if s_vals is not None else None
    gr = torch.empty((1, plan.n), dtype=torch.complex128, device=dev)
    gl = torch.empty_like(gr) if config.compute_gless else None
    ws = plan.workspace(1, config.compute_gless, dev)
    plan.run(a_d, s_d, gr, gl, config.compute_gless, config.pivot_rtol, ws=ws, groups=(0, plan.first_down_group),
             sigma_sym=ssym)
    plan.check_status(ws, 1)
    oa, oo, _ = _elim_layout(plan)
    arenas = [x.cpu().numpy() for x in _arena_views(plan, ws)]
    data: dict[int, ClusterData] = {}
    for k in np.nonzero((plan.kind == 0) | (plan.kind == 1))[0]:
        if oa[k] < 0:
            continue
        label = int(plan.label[k])
        bset = plan.cluster_set(label, 1)
        b = int(plan.b[k])
        off = int(oo[k])
        up = arenas[int(oa[k])]
        u = up[off:off + b * b].reshape(b, b).copy()
        r = up[off + b * b:off + 2 * b * b].reshape(b, b).copy() if config.compute_gless else None
        data[label] = ClusterData(DenseBlock(bset, bset, u), DenseBlock(bset, bset, r) if r is not None else None)
    _charge(ledger, plan, (plan.kind == 0) | (plan.kind == 1), config, herm)
    return data


def downward_pass(tree, a: SparseOperator, sigma: SparseOperator | None, cluster_data: dict, config,
                  ledger: FlopLedger | None = None, engine=None, leaf_callback=None,
                  keep_all: bool = True) -> dict[int, ClusterData]:
    """solver.py:311-375: complement-cluster elimination root-to-leaves from the given upward
    ``cluster_data``; returns {-label: ClusterData} (the root's complement is empty).
    ``leaf_callback(leaf, neg_data)`` fires for every leaf in the reference's DFS order;
    with ``keep_all`` False only the callback sees the complement data."""
    import torch

    from .mesh import annotated_tree

    plan, am = _plan_for_tree(tree, a)
    dev = _dev()
    a_vals, s_vals, ssym, herm = _values(plan, am, sigma, config.compute_gless)
    a_d = torch.from_numpy(a_vals).to(dev)
    s_d = torch.from_numpy(s_vals).to(dev) if s_vals is not None else None
    gr = torch.empty((1, plan.n), dtype=torch.complex128, device=dev)
    gl = torch.empty_like(gr) if config.compute_gless else None
    ws = plan.workspace(1, config.compute_gless, dev)
    oa, oo, _ = _elim_layout(plan)
    arenas = _arena_views(plan, ws)
    # the caller's upward blocks into the upward arena (the slots the downward merges read)
    up_host = np.zeros(arenas[0].numel(), np.complex128)
    for k in np.nonzero(((plan.kind == 0) | (plan.kind == 1)) & (oa == 0))[0]:
        label = int(plan.label[k])
        if label not in cluster_data:
            raise TreeStateError(f"cluster_data has no entry for cluster {label}")
        cd = cluster_data[label]
        b = int(plan.b[k])
        off = int(oo[k])
        if cd.u.values.shape != (b, b):
            raise ValueError(f"cluster {label}: U block shape {cd.u.values.shape} != ({b}, {b})")
        up_host[off:off + b * b] = cd.u.values.ravel()
        if config.compute_gless:
            if cd.r is None:
                raise ValueError(f"cluster {label}: compute_gless needs its R block")
            up_host[off + b * b:off + 2 * b * b] = cd.r.values.ravel()
    arenas[0].copy_(torch.from_numpy(up_host).to(dev))
    data: dict[int, ClusterData] = {}
    g = plan.groups
    start = np.concatenate([[0], np.cumsum(g["count"])])
    for gi in range(plan.first_down_group, len(g["count"])):
        if int(g["pass"][gi]) != 1:
            continue  # final leaf steps belong to the extraction
        plan.run(a_d, s_d, gr, gl, config.compute_gless, config.pivot_rtol, ws=ws, groups=(gi, gi + 1),
                 sigma_sym=ssym)
        plan.check_status(ws, 1)
        for k in range(int(start[gi]), int(start[gi + 1])):
            if plan.kind[k] != 2 or oa[k] < 0:
                continue
            b = int(plan.b[k])
            off = int(oo[k])
            blk = arenas[int(oa[k])][off:off + 2 * b * b].cpu().numpy()
            label = int(plan.label[k])  # negative: complement label
            bset = plan.cluster_set(-label, 3)
            data[label] = ClusterData(DenseBlock(bset, bset, blk[:b * b].reshape(b, b).copy()),
                                      DenseBlock(bset, bset, blk[b * b:].reshape(b, b).copy())
                                      if config.compute_gless else None)
    empty = DenseBlock(np.array([], np.int64), np.array([], np.int64), np.zeros((0, 0)))
    data[-1] = ClusterData(empty, empty if config.compute_gless else None)
    _charge(ledger, plan, plan.kind == 2, config, herm)
    if leaf_callback is not None:
        atree, _ = annotated_tree(plan)
        stack = [atree.root]
        while stack:  # the reference's DFS order (solver.py:362-371)
            c = stack.pop()
            if c.is_leaf:
                leaf_callback(c, data[-c.label])
            else:
                stack.extend(reversed(c.children))
    if not keep_all:
        return {-1: data[-1]}
    return data


# ------------------------------------------------------------------------------ leaf extraction
def _final(a, sigma, leaf, ring, neg, ledger, want_sigma, pivot_rtol):
    """solver.py:392-418: U_f and R_f of one leaf from its complement data (device)."""
    nodes = np.asarray(leaf.nodes, np.int64)
    ring = np.asarray(ring, np.int64)
    sig = None
    if want_sigma:
        sig = (neg.r.values, _extract(sigma, ring, nodes), _extract(sigma, nodes, ring), _extract(sigma, nodes, nodes))
    try:
        u_f, r_f, _ = _device_elimination(neg.u.values, _extract(a, ring, nodes), _extract(a, nodes, ring),
                                          _extract(a, nodes, nodes), sig, pivot_rtol)
    except SingularPivotError as exc:
        if exc.node is not None and exc.node < ring.size:
            exc.node = int(ring[exc.node])
        exc.cluster = leaf.label
        raise
    t, c = ring.size, nodes.size
    if ledger is not None:
        if t:
            ledger.add("naive_dense", flop_model("naive_dense", s=t, b=c))
            if want_sigma:
                ledger.add("sigma_naive", flop_model("sigma_naive", s=t, b=c))
    return u_f, r_f


def leaf_extract_gr(leaf, a: SparseOperator, neg: ClusterData, ring, ledger: FlopLedger | None = None,
                    pivot_rtol: float = 1e-12) -> DenseBlock:
    """solver.py:421-432: full inverse block over one leaf cluster from its complement data."""
    ledger = ledger if ledger is not None else FlopLedger()
    u_f, _ = _final(a, None, leaf, ring, neg, ledger, False, pivot_rtol)
    g = _device_inverse(u_f, leaf.label)
    ledger.add("dense_inverse", flop_model("dense_inverse", c=g.shape[0]))
    return DenseBlock(leaf.nodes, leaf.nodes, g.cpu().numpy())


def leaf_extract_gless(leaf, a: SparseOperator, sigma: SparseOperator, neg: ClusterData, ring,
                       ledger: FlopLedger | None = None, pivot_rtol: float = 1e-12) -> DenseBlock:
    """solver.py:435-451: G^<(C, C) = G R_f G^H over one leaf."""
    ledger = ledger if ledger is not None else FlopLedger()
    u_f, r_f = _final(a, sigma, leaf, ring, neg, ledger, True, pivot_rtol)
    g = _device_inverse(u_f, leaf.label)
    ledger.add("dense_inverse", flop_model("dense_inverse", c=g.shape[0]))
    gless = (g @ r_f) @ g.conj().T
    ledger.add("gless_sandwich", flop_model("gless_sandwich", c=g.shape[0]))
    return DenseBlock(leaf.nodes, leaf.nodes, gless.cpu().numpy())


def leaf_extract_offdiag(leaf, a: SparseOperator, neg: ClusterData, ring, g: np.ndarray,
                         ledger: FlopLedger | None = None) -> dict:
    """solver.py:454-484: inverse entries between the leaf and its adjacent set (one
    back-substitution each way), stencil-adjacent pairs only; pairs inside the leaf from g."""
    import torch

    ledger = ledger if ledger is not None else FlopLedger()
    nodes = np.asarray(leaf.nodes, np.int64)
    ring = np.asarray(ring, np.int64)
    out = {}
    adjacency = a.adjacency()
    g = np.asarray(g, np.complex128)
    sub = adjacency[nodes][:, nodes].tocoo()
    for i, j in zip(sub.row, sub.col):
        out[(int(nodes[i]), int(nodes[j]))] = complex(g[i, j])
    if ring.size:
        dev = _dev()
        gd = torch.from_numpy(g).to(dev)
        a_bc = torch.from_numpy(_extract(a, ring, nodes)).to(dev)
        a_cb = torch.from_numpy(_extract(a, nodes, ring)).to(dev)
        u_ring = neg.u.values
        c = nodes.size
        zero = np.zeros((c, c), np.complex128)
        # G(ring, C) = -U^-1 (A_rC g): L = Abs Ass^-1 with Ass = U^T, Abs = (A_rC g)^T gives L^T = U^-1 A_rC g
        _, _, l1 = _device_elimination(u_ring.T, np.zeros((ring.size, c), np.complex128), (a_bc @ gd).T, zero,
                                       rtol=_TINY, want_l=True)
        g_bc = -(l1.T)
        # G(C, ring) = -(g A_Cr) U^-1: L = Abs Ass^-1 with Ass = U, Abs = g A_Cr
        _, _, l2 = _device_elimination(u_ring, np.zeros((ring.size, c), np.complex128), gd @ a_cb, zero, rtol=_TINY,
                                       want_l=True)
        g_cb = -l2
        ledger.add("offdiag_backsub", flop_model("offdiag_backsub", t=ring.size, c=nodes.size))
        g_bc = g_bc.cpu().numpy()
        g_cb = g_cb.cpu().numpy()
        cross = adjacency[ring][:, nodes].tocoo()
        for i, j in zip(cross.row, cross.col):
            u, v = int(ring[i]), int(nodes[j])
            out[(u, v)] = complex(g_bc[i, j])
            out[(v, u)] = complex(g_cb[j, i])
    return out
