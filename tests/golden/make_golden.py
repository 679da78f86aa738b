"""Generate golden vectors from the REFERENCE implementation (run in the build
container only; /root/reference does not exist on the GPU box).

    python tests/golden/make_golden.py

Imports find_selinv read-only from /root/reference/pkg/src and writes small
.npz fixtures next to this script.  The GPU tests and the oracle tests compare
against these files.
"""

import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
sys.path.insert(0, "/root/reference/pkg/src")

import find_selinv as ref  # noqa: E402
from find_selinv.mesh import annotate_boundaries, build_cluster_tree, complement_boundary_sets  # noqa: E402
from find_selinv.operators import SparseOperator  # noqa: E402
from find_selinv.oracle import dense_gless_diag, dense_gr_diag  # noqa: E402

from paper_1104_0623_b200.configs import build_problem, config_problem  # noqa: E402


def frac(x):
    return np.array([x.numerator, x.denominator], dtype=object)


def ledger_arrays(led):
    keys = sorted(led.by_kernel)
    return np.array(keys), np.array([[v.numerator, v.denominator] for v in (led.by_kernel[k] for k in keys)], dtype=object)


def solve_ref(nx, ny, a_csr, s_csr, kernel="naive", leaf_max=2, compute_gless=True):
    res = ref.solve(ref.Mesh(nx, ny), SparseOperator(a_csr), SparseOperator(s_csr) if s_csr is not None else None,
                    ref.SolverConfig(kernel=kernel, compute_gless=compute_gless, leaf_max=leaf_max))
    return res


def contact_cases():
    """cfg0 itself plus reduced-size variants of the BASELINE generator."""
    cases = {
        "cfg0": (config_problem(0), 0),
        "c5_16x12": (build_problem(16, 12, [0.7, 2.9], seed=11, stencil=5, vamp=0.5), None),
        "c9_20x20": (build_problem(20, 20, [1.3], seed=12, stencil=9, vamp=0.5), None),
        "c5_8x30": (build_problem(8, 30, [0.5, 3.5], seed=13, stencil=5, vamp=1.0), None),
    }
    for name, (p, _) in cases.items():
        gr, gl, W = [], [], []
        led_keys = None
        for k in range(p.energies.size):
            a = p.a_csr(k)
            s = p.sigma_csr()
            r = solve_ref(p.nx, p.ny, a, s)
            gr.append(r.gr_diag)
            gl.append(r.gless_diag)
            W = r.ledger.multiplications
            if p.n <= 2500:
                dg = dense_gr_diag(a.toarray())
                dl = dense_gless_diag(a.toarray(), s.toarray())
                print(name, k, "ref vs dense", np.abs(r.gr_diag - dg).max() / np.abs(dg).max(),
                      np.abs(r.gless_diag - dl).max() / np.abs(dl).max())
        extra = {}
        for kern in ("parallel_inverse", "sequential_inverse", "block_lu", "naive_lu"):
            if p.n <= 400:
                r = solve_ref(p.nx, p.ny, p.a_csr(0), p.sigma_csr(), kernel=kern)
                extra[f"W_{kern}"] = frac(r.ledger.multiplications)
                extra[f"stats_up_{kern}"] = np.array(r.stats["upward_exception_entries"])
                extra[f"stats_down_{kern}"] = np.array(r.stats["downward_exception_entries"])
        np.savez_compressed(HERE / f"{name}.npz", nx=p.nx, ny=p.ny, indptr=p.indptr, indices=p.indices,
                            h_vals=p.h_vals, diag_pos=p.diag_pos, s_vals=p.s_vals, energies=p.energies,
                            gr=np.array(gr), gl=np.array(gl), W=frac(W), allow_pickle=True, **extra)
        print("wrote", name, p.n, "W", W)


def stencil_cases():
    """The reference test-suite generators (pkg/tests/conftest.py:11-78), restated."""
    out = {}
    rng_cases = [(6, 4, 10, 11, "stencil"), (4, 4, 7, 8, "diagonal"), (8, 8, 15, 16, "stencil"), (3, 5, 21, 22, "diagonal"),
                 (16, 16, 1000, 1001, "diagonal"), (5, 7, 31, 32, "stencil")]
    for nx, ny, sa, ss, mode in rng_cases:
        mesh = ref.build_mesh(nx, ny)
        rng = np.random.default_rng(sa)
        adj = mesh.adjacency().tocoo()
        mask = adj.row < adj.col
        rows, cols = adj.row[mask], adj.col[mask]
        m = rows.size
        degree = np.asarray(mesh.adjacency().sum(axis=1)).ravel()
        hop = rng.standard_normal(m) + 1j * rng.standard_normal(m)
        back = rng.standard_normal(m) + 1j * rng.standard_normal(m)
        diag = degree * 1.6 + 1.0 + rng.random(mesh.n) + 1j * (1.0 + rng.random(mesh.n))
        ids = np.arange(mesh.n)
        a = SparseOperator.from_coo(mesh.n, np.concatenate([ids, rows, cols]), np.concatenate([ids, cols, rows]),
                                    np.concatenate([diag.astype(complex), hop, back]))
        rng2 = np.random.default_rng(ss)
        if mode == "diagonal":
            vals = rng2.standard_normal(mesh.n) + 1j * rng2.standard_normal(mesh.n)
            s = SparseOperator.from_coo(mesh.n, ids, ids, vals)
        else:
            h2 = rng2.standard_normal(m) + 1j * rng2.standard_normal(m)
            b2 = rng2.standard_normal(m) + 1j * rng2.standard_normal(m)
            d2 = rng2.standard_normal(mesh.n) + 1j * rng2.standard_normal(mesh.n)
            s = SparseOperator.from_coo(mesh.n, np.concatenate([ids, rows, cols]), np.concatenate([ids, cols, rows]),
                                        np.concatenate([d2, h2, b2]))
        res = {}
        for lm in (1, 2, 3):
            r = ref.solve(mesh, a, s, ref.SolverConfig(kernel="naive", compute_gless=True, leaf_max=lm))
            res[f"gr_{lm}"] = r.gr_diag
            res[f"gl_{lm}"] = r.gless_diag
            res[f"W_{lm}"] = frac(r.ledger.multiplications)
        am, sm = a.matrix, s.matrix
        np.savez_compressed(HERE / f"stencil_{nx}x{ny}.npz", nx=nx, ny=ny, a_data=am.data, a_indices=am.indices,
                            a_indptr=am.indptr, s_data=sm.data, s_indices=sm.indices, s_indptr=sm.indptr,
                            dense_gr=dense_gr_diag(a.to_dense()), dense_gl=dense_gless_diag(a.to_dense(), s.to_dense()),
                            allow_pickle=True, **res)
        print("wrote stencil", nx, ny)


def set_cases():
    """Per-cluster node sets from the reference (mesh.py:209-290) for plan validation."""
    for name, p in {"sets_c5_12x10": build_problem(12, 10, [1.0], seed=5, stencil=5),
                    "sets_c9_9x14": build_problem(9, 14, [1.0], seed=6, stencil=9)}.items():
        a = SparseOperator(p.a_csr(0))
        for lm in (1, 2, 3):
            tree = build_cluster_tree(ref.Mesh(p.nx, p.ny), lm)
            annotate_boundaries(tree, a.adjacency())
            comps = complement_boundary_sets(tree, a.adjacency())
            labels, sets = [], []
            for c in sorted(tree.by_label.values(), key=lambda c: c.label):
                labels.append(c.label)
                sets.append([c.nodes, c.boundary, c.private_inner, comps[-c.label].boundary, comps[-c.label].private_inner])
            flat, offs = [], [0]
            for row in sets:
                for arr in row:
                    flat.append(np.asarray(arr, np.int64))
                    offs.append(offs[-1] + len(arr))
            np.savez_compressed(HERE / f"{name}_lm{lm}.npz", nx=p.nx, ny=p.ny, indptr=p.indptr, indices=p.indices,
                                labels=np.array(labels), flat=np.concatenate(flat), offs=np.array(offs))
        print("wrote", name)


def _ref_extended_gless(mesh, a, s, leaf_max):
    """G^< on every directed adjacent pair, from the reference's own ring+leaf
    extraction (_extended_extraction, solver.py:487-507) run on each leaf in the
    downward DFS, keeping the pairs full-leaves extraction owns (first writer,
    solver.py:666-669): pairs inside the leaf and between the leaf and its ring."""
    from find_selinv import solver as rs

    cfg = ref.SolverConfig(kernel="naive", compute_gless=True, leaf_max=leaf_max)
    tree = build_cluster_tree(mesh, leaf_max)
    adj = a.adjacency()
    annotate_boundaries(tree, adj)
    comps = complement_boundary_sets(tree, adj)
    led = ref.FlopLedger()
    engine = rs._Engine(a, s, tree, comps, cfg, led)
    pos = rs.upward_pass(tree, a, s, cfg, engine=engine)
    out = {}

    def on_leaf(leaf, neg):
        g_t, gl_t, labels = rs._extended_extraction(engine, leaf, neg, True)
        t = labels.size - leaf.nodes.size
        region = adj[labels][:, labels].tocoo()
        for i, j in zip(region.row, region.col):
            if i < t and j < t:
                continue  # ring-ring pairs belong to other leaves under full-leaves
            key = (int(labels[i]), int(labels[j]))
            if key not in out:
                out[key] = complex(gl_t[i, j])

    rs.downward_pass(tree, a, s, pos, cfg, engine=engine, leaf_callback=on_leaf, keep_all=False)
    return out


def offdiag_cases():
    """Off-diagonal G^r (reference solve, compute_offdiag, both tilings) and G^< (reference
    _extended_extraction) on contact-style and general-Sigma problems."""
    cases = {
        "off_c5_10x8": (build_problem(10, 8, [0.9, 2.2], seed=21, stencil=5), 2, False),
        "off_c9_9x7": (build_problem(9, 7, [1.7], seed=22, stencil=9), 2, False),
        "off_c5_7x9_lm3": (build_problem(7, 9, [1.1], seed=23, stencil=5), 3, False),
        "off_gen_8x8": (build_problem(8, 8, [1.4], seed=24, stencil=5), 2, True),
    }
    for name, (p, lm, general) in cases.items():
        mesh = ref.Mesh(p.nx, p.ny)
        s_csr = p.sigma_csr()
        if general:  # a non-Hermitian Sigma on the same pattern: exercises the general G^< path
            rng = np.random.default_rng(99)
            s_csr = s_csr.copy()
            s_csr.data = s_csr.data + 0.3 * (rng.standard_normal(s_csr.nnz) + 1j * rng.standard_normal(s_csr.nnz))
        pairs = None
        gr_full, gr_half, gl_ext = [], [], []
        led = {}
        for k in range(p.energies.size):
            a_op = SparseOperator(p.a_csr(k))
            s_op = SparseOperator(s_csr)
            rf = ref.solve(mesh, a_op, s_op, ref.SolverConfig(kernel="naive", compute_gless=True, compute_offdiag=True,
                                                              leaf_max=lm))
            rh = ref.solve(mesh, a_op, s_op, ref.SolverConfig(kernel="naive", compute_gless=True, compute_offdiag=True,
                                                              tiling="half-leaves", leaf_max=lm))
            if pairs is None:
                pairs = np.array(sorted(rf.offdiag), dtype=np.int64)
                led = {"W_full": frac(rf.ledger.multiplications), "W_half": frac(rh.ledger.multiplications)}
            gr_full.append([rf.offdiag[tuple(q)] for q in pairs.tolist()])
            gr_half.append([rh.offdiag[tuple(q)] for q in pairs.tolist()])
            ext = _ref_extended_gless(mesh, a_op, s_op, lm)
            gl_ext.append([ext[tuple(q)] for q in pairs.tolist()])
            A = a_op.to_dense()
            G = np.linalg.inv(A)
            GL = G @ s_op.to_dense() @ G.conj().T
            print(name, k, "ref gr vs dense", np.abs(np.array(gr_full[-1]) - G[pairs[:, 0], pairs[:, 1]]).max(),
                  "ext gl vs dense", np.abs(np.array(gl_ext[-1]) - GL[pairs[:, 0], pairs[:, 1]]).max())
        np.savez_compressed(HERE / f"{name}.npz", nx=p.nx, ny=p.ny, leaf_max=lm, indptr=p.indptr, indices=p.indices,
                            h_vals=p.h_vals, diag_pos=p.diag_pos, s_data=s_csr.data, s_indices=s_csr.indices,
                            s_indptr=s_csr.indptr, energies=p.energies, pairs=pairs, gr_full=np.array(gr_full),
                            gr_half=np.array(gr_half), gl_ext=np.array(gl_ext), allow_pickle=True, **led)
        print("wrote", name, pairs.shape[0], "pairs")


def io_cases():
    """Matrix Market files written by the reference (operators.py:222-230) and its CSV
    exports (solver.py:709-734) of one reference result, for byte-level format checks."""
    from find_selinv.operators import write_matrix_market
    from find_selinv.solver import diag_to_csv, offdiag_to_csv

    p = build_problem(6, 5, [1.2], seed=41, stencil=5)
    mesh = ref.Mesh(p.nx, p.ny)
    a = SparseOperator(p.a_csr(0))
    s = SparseOperator(p.sigma_csr())
    write_matrix_market(HERE / "io_a_mesh.mtx", a, mesh)
    write_matrix_market(HERE / "io_a_plain.mtx", a)
    r = ref.solve(mesh, a, s, ref.SolverConfig(compute_gless=True, compute_offdiag=True))
    keys = np.array(sorted(r.offdiag), dtype=np.int64)
    np.savez_compressed(HERE / "io_csv.npz", nx=p.nx, ny=p.ny, gr=r.gr_diag, gl=r.gless_diag, off_keys=keys,
                        off_vals=np.array([r.offdiag[tuple(k)] for k in keys.tolist()]),
                        diag_csv=np.array(diag_to_csv(r, mesh)), offdiag_csv=np.array(offdiag_to_csv(r)))
    r2 = ref.solve(mesh, a, None, ref.SolverConfig(compute_gless=False))
    np.savez_compressed(HERE / "io_csv_nogless.npz", gr=r2.gr_diag, diag_csv=np.array(diag_to_csv(r2, mesh)),
                        offdiag_csv=np.array(offdiag_to_csv(r2)))
    print("wrote io cases")


def rgf_cases():
    """Reference RGF (rgf.py:118-208) diagonals and ledgers on contact and stencil problems."""
    from find_selinv.rgf import block_partition, rgf_gless_diag, rgf_gr_diag

    cases = {"rgf_c5_12x9": build_problem(12, 9, [0.8, 2.3], seed=51, stencil=5),
             "rgf_c9_10x8": build_problem(10, 8, [1.6], seed=52, stencil=9)}
    for name, p in cases.items():
        mesh = ref.Mesh(p.nx, p.ny)
        s_op = SparseOperator(p.sigma_csr())
        gr, gl = [], []
        for k in range(p.energies.size):
            a_op = SparseOperator(p.a_csr(k))
            bt, sbt = block_partition(a_op, mesh), block_partition(s_op, mesh)
            lg, ll = ref.FlopLedger(), ref.FlopLedger()
            gr.append(rgf_gr_diag(bt, lg))
            gl.append(rgf_gless_diag(bt, sbt, ll))
        np.savez_compressed(HERE / f"{name}.npz", nx=p.nx, ny=p.ny, indptr=p.indptr, indices=p.indices,
                            h_vals=p.h_vals, diag_pos=p.diag_pos, s_vals=p.s_vals, energies=p.energies,
                            gr=np.array(gr), gl=np.array(gl), W_gr=frac(lg.multiplications),
                            W_gl=frac(ll.multiplications), allow_pickle=True)
        print("wrote", name, "W_gr", lg.multiplications, "W_gl", ll.multiplications)


if __name__ == "__main__":
    import sys as _sys

    if "rgf" in _sys.argv:
        rgf_cases()
    elif "io" in _sys.argv:
        io_cases()
    elif "offdiag" in _sys.argv:
        offdiag_cases()
    else:
        set_cases()
        stencil_cases()
        contact_cases()
        offdiag_cases()
        io_cases()
        rgf_cases()
