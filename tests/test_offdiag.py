"""Off-diagonal extraction (SolverConfig.compute_offdiag; solver.py:454-484, 637-642, 666-669)
and the G^< cross blocks (the reference's _extended_extraction, solver.py:487-507).

Golden vectors (tests/golden/off_*.npz, tests/golden/make_golden.py offdiag_cases) come from
the reference itself: G^r pairs from ``solve(..., compute_offdiag=True)`` under both tilings,
G^< pairs from ``_extended_extraction`` run leaf by leaf with full-leaves ownership.
Tolerance: max|Δ|/max|ref| <= 1e-10 (BASELINE.json north star)."""

import numpy as np
import pytest
import scipy.sparse as sp

from conftest import golden_frac, load_golden

OFF_CASES = ["off_c5_10x8", "off_c9_9x7", "off_c5_7x9_lm3", "off_gen_8x8"]
TOL = 1e-10


def rel(x, ref):
    return float(np.max(np.abs(np.asarray(x) - np.asarray(ref))) / np.max(np.abs(ref)))


def golden_ops(g, k):
    from paper_1104_0623_b200.configs import DeviceProblem

    nx, ny = int(g["nx"]), int(g["ny"])
    n = nx * ny
    s_csr = sp.csr_matrix((g["s_data"], g["s_indices"], g["s_indptr"]), shape=(n, n))
    p = DeviceProblem(nx, ny, g["indptr"], g["indices"], g["h_vals"], g["diag_pos"], np.zeros(g["indices"].size, complex),
                      g["energies"])
    return p, p.a_csr(k), s_csr


# ------------------------------------------------------------------ CPU: oracle + plan + ledger
@pytest.mark.parametrize("name", OFF_CASES)
def test_oracle_offdiag_matches_reference(name):
    from oracle.find_oracle import FindOracle

    g = load_golden(name)
    pairs = [tuple(q) for q in g["pairs"].tolist()]
    for k in range(g["energies"].size):
        p, a, s = golden_ops(g, k)
        r = FindOracle(p.nx, p.ny, a, leaf_max=int(g["leaf_max"])).solve(a, s, compute_offdiag=True)
        assert set(r.offdiag) == set(pairs)
        assert rel([r.offdiag[q] for q in pairs], g["gr_full"][k]) < 1e-12
        assert rel([r.offdiag_gless[q] for q in pairs], g["gl_ext"][k]) < 1e-12


@pytest.mark.parametrize("name", OFF_CASES)
def test_offdiag_pairs_match_reference(name):
    from paper_1104_0623_b200.plan import plan_for

    g = load_golden(name)
    plan, _ = plan_for(int(g["nx"]), int(g["ny"]), g["indptr"], g["indices"], int(g["leaf_max"]))
    assert np.array_equal(plan.offdiag_pairs(), g["pairs"])


@pytest.mark.parametrize("name", OFF_CASES)
def test_offdiag_ledger_matches_reference(name):
    import warnings

    from paper_1104_0623_b200 import SolverConfig
    from paper_1104_0623_b200.plan import plan_for
    from paper_1104_0623_b200.solver import _ledger_cached

    g = load_golden(name)
    lm = int(g["leaf_max"])
    plan, _ = plan_for(int(g["nx"]), int(g["ny"]), g["indptr"], g["indices"], lm)
    full = _ledger_cached(plan, SolverConfig(compute_offdiag=True, leaf_max=lm), False)
    assert full.multiplications == golden_frac(g["W_full"])
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        half = _ledger_cached(plan, SolverConfig(compute_offdiag=True, tiling="half-leaves", leaf_max=lm), False)
    assert half.multiplications == golden_frac(g["W_half"])


def test_half_leaves_selection_rules():
    """select_tiling (solver.py:522-556): boundary leaves plus a checkerboard of the interior."""
    from paper_1104_0623_b200.plan import plan_for
    from paper_1104_0623_b200.solver import _leaf_table, half_leaves_selection
    from paper_1104_0623_b200.configs import build_problem

    p = build_problem(16, 16, [1.0], seed=1)
    plan, _ = plan_for(p.nx, p.ny, p.indptr, p.indices)
    sel = half_leaves_selection(plan)
    _, rect = _leaf_table(plan)
    assert sel.size == 64 and sel.sum() == 28 + 18  # 28 boundary tiles + half of the 6x6 interior
    ti, tj = rect[:, 0] // 2, rect[:, 1] // 2
    assert np.all(sel[(ti == 0) | (tj == 0) | (ti == 7) | (tj == 7)])
    q = build_problem(12, 12, [1.0], seed=1)  # 12 -> 6 -> 3 -> {2, 1}: non-uniform leaves fall back
    plan2, _ = plan_for(q.nx, q.ny, q.indptr, q.indices)
    with pytest.warns(UserWarning):
        assert half_leaves_selection(plan2) is None


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
@pytest.mark.parametrize("name", OFF_CASES)
@pytest.mark.parametrize("tiling", ["full-leaves", "half-leaves"])
def test_offdiag_matches_reference_golden(cuda, name, tiling):
    import warnings

    from paper_1104_0623_b200 import Mesh, SolverConfig, SparseOperator, solve

    g = load_golden(name)
    pairs = [tuple(q) for q in g["pairs"].tolist()]
    for k in range(g["energies"].size):
        p, a, s = golden_ops(g, k)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            res = solve(Mesh(p.nx, p.ny), SparseOperator(a), SparseOperator(s),
                        SolverConfig(compute_offdiag=True, tiling=tiling, leaf_max=int(g["leaf_max"])))
        assert set(res.offdiag) == set(pairs)
        want = g["gr_full"][k] if tiling == "full-leaves" else g["gr_half"][k]
        assert rel([res.offdiag[q] for q in pairs], want) < TOL
        assert rel([res.offdiag_gless[q] for q in pairs], g["gl_ext"][k]) < TOL
        assert res.ledger.multiplications == golden_frac(g["W_full" if tiling == "full-leaves" else "W_half"])


def _dense_check(res_gr, res_gl, pairs, a, s):
    G = np.linalg.inv(a.toarray())
    GL = G @ s.toarray() @ G.conj().T
    u, v = pairs[:, 0], pairs[:, 1]
    assert rel(res_gr, G[u, v]) < TOL
    if res_gl is not None:
        assert rel(res_gl, GL[u, v]) < TOL


@pytest.mark.gpu
@pytest.mark.parametrize("general", [False, True])
def test_offdiag_cta_path_vs_dense(cuda, general):
    """Contact rows of 80 nodes: leaf rings of ~80 run the blocked CTA path, whose
    factorization the off-diagonal kernel reuses; checked against dense inversion."""
    from paper_1104_0623_b200 import Mesh, SolverConfig, SparseOperator, solve_batch
    from paper_1104_0623_b200.configs import build_problem
    from paper_1104_0623_b200.plan import plan_for

    p = build_problem(80, 18, [0.8, 2.6], seed=31, stencil=5)
    s = p.sigma_csr()
    if general:
        rng = np.random.default_rng(5)
        s = s.copy()
        s.data = s.data + 0.2 * (rng.standard_normal(s.nnz) + 1j * rng.standard_normal(s.nnz))
    plan, _ = plan_for(p.nx, p.ny, p.indptr, p.indices)
    fin = plan.kind == 3
    assert (plan.s[fin] + plan.b[fin]).max() > 64  # CTA-path final steps present
    ops = [SparseOperator(p.a_csr(k)) for k in range(2)]
    res = solve_batch(Mesh(p.nx, p.ny), ops, SparseOperator(s), SolverConfig(compute_offdiag=True))
    for k in range(2):
        _dense_check(res.offdiag_gr[k], res.offdiag_gless[k], res.offdiag_pairs, p.a_csr(k), s)


@pytest.mark.gpu
def test_offdiag_gr_only_and_diag_unchanged(cuda):
    from paper_1104_0623_b200 import Mesh, SolverConfig, SparseOperator, solve
    from paper_1104_0623_b200.configs import build_problem

    p = build_problem(20, 16, [1.9], seed=4, stencil=9)
    a, s = p.a_csr(0), p.sigma_csr()
    r0 = solve(Mesh(p.nx, p.ny), SparseOperator(a), SparseOperator(s), SolverConfig())
    r1 = solve(Mesh(p.nx, p.ny), SparseOperator(a), None, SolverConfig(compute_gless=False, compute_offdiag=True))
    assert r1.offdiag_gless is None and r1.gless_diag is None
    assert np.array_equal(r0.gr_diag, r1.gr_diag)
    pairs = np.array(sorted(r1.offdiag), dtype=np.int64)
    _dense_check([r1.offdiag[tuple(q)] for q in pairs.tolist()], None, pairs, a, s)
    assert "offdiag_backsub" in r1.ledger.by_kernel


@pytest.mark.gpu
def test_offdiag_diagonal_operator_is_empty(cuda):
    """test_solver.py:136-142: no adjacency, nothing to report."""
    from paper_1104_0623_b200 import Mesh, SolverConfig, SparseOperator, solve

    n = 12
    a = SparseOperator(sp.csr_matrix(sp.diags(np.arange(1, n + 1) + 1j)))
    res = solve(Mesh(4, 3), a, None, SolverConfig(compute_gless=False, compute_offdiag=True))
    assert res.offdiag == {}


@pytest.mark.gpu
@pytest.mark.parametrize("nx,ny", [(1, 1), (2, 2), (1, 9), (7, 1), (3, 5)])
def test_offdiag_degenerate_meshes_vs_dense(cuda, nx, ny):
    from conftest import stencil_operator, stencil_sigma

    from paper_1104_0623_b200 import SolverConfig, solve

    mesh, a = stencil_operator(nx, ny, seed=nx * 10 + ny)
    s = stencil_sigma(mesh, seed=3, mode="stencil")
    res = solve(mesh, a, s, SolverConfig(compute_offdiag=True))
    pairs = np.array(sorted(res.offdiag), dtype=np.int64).reshape(-1, 2)
    if pairs.size:
        _dense_check([res.offdiag[tuple(q)] for q in pairs.tolist()],
                     [res.offdiag_gless[tuple(q)] for q in pairs.tolist()], pairs, a.matrix, s.matrix)


@pytest.mark.gpu
def test_cfg3_offdiag_full_scale_against_sparse_lu(cuda):
    """BASELINE config 3 (256 x 1024, V ~ U[-1,1]) at full size, two of its energy points:
    G^r and G^< on sampled adjacent pairs (stencil and contact-row pairs) against
    independent sparse-LU solves x_i = A^-H e_i: G_ij = conj(x_i[j]), G^<_ij = x_i^H S x_j."""
    import scipy.sparse.linalg as spla

    from paper_1104_0623_b200 import Mesh, SolverConfig, SparseOperator, solve_batch
    from paper_1104_0623_b200.configs import CONFIGS, build_problem

    c = CONFIGS[3]
    energies = np.asarray(c.energies)[[0, len(c.energies) - 1]]
    p = build_problem(c.nx, c.ny, energies, seed=3, stencil=c.stencil, vamp=c.vamp)
    sig = p.sigma_csr()
    res = solve_batch(Mesh(p.nx, p.ny), [SparseOperator(p.a_csr(k)) for k in range(2)], SparseOperator(sig),
                      SolverConfig(compute_offdiag=True))
    pairs = res.offdiag_pairs
    rng = np.random.default_rng(3)
    pick = list(rng.choice(pairs.shape[0], 10, replace=False))
    pick += list(np.nonzero((pairs[:, 0] < p.nx) & (pairs[:, 1] < p.nx))[0][[0, 777]])  # contact row (iy = 0)
    pick += list(np.nonzero((pairs[:, 0] >= p.n - p.nx) & (pairs[:, 1] < p.n - p.nx))[0][:2])
    for k in range(2):
        lu = spla.splu(p.a_csr(k).conj().T.tocsc())
        cache = {}

        def x_of(i):
            if i not in cache:
                e = np.zeros(p.n, complex)
                e[i] = 1.0
                cache[i] = lu.solve(e)
            return cache[i]

        scale_r = np.max(np.abs(res.gr_diag[k]))
        scale_l = np.max(np.abs(res.gless_diag[k]))
        for q in pick:
            i, j = map(int, pairs[q])
            xi, xj = x_of(i), x_of(j)
            assert abs(res.offdiag_gr[k, q] - np.conj(xi[j])) < 1e-10 * scale_r
            assert abs(res.offdiag_gless[k, q] - np.vdot(xi, sig @ xj)) < 1e-10 * scale_l
