"""GPU RGF (rgf.py:1-208 restated on the device, batched over energy points) against the
reference's own RGF outputs and ledgers (tests/golden/rgf_*.npz, make_golden.py rgf_cases),
dense inversion and the FIND path."""

import numpy as np
import pytest

from conftest import golden_frac, load_golden, problem_from_golden

RGF_CASES = ["rgf_c5_12x9", "rgf_c9_10x8"]


def rel(x, ref):
    return float(np.max(np.abs(np.asarray(x) - np.asarray(ref))) / np.max(np.abs(ref)))


def test_block_partition_round_trip():
    """rgf.py:43-72: line blocks reassemble the operator; non-tridiagonal patterns are rejected."""
    import scipy.sparse as sp

    from paper_1104_0623_b200 import Mesh, SparseOperator
    from paper_1104_0623_b200.configs import build_problem
    from paper_1104_0623_b200.rgf import block_partition

    p = build_problem(6, 5, [1.0], seed=3, stencil=9)
    a = p.a_csr(0)
    bt = block_partition(SparseOperator(a), Mesh(p.nx, p.ny))
    assert bt.num_blocks == 5
    full = sp.block_diag(bt.diag).toarray()
    for i in range(4):
        full[i * 6:(i + 1) * 6, (i + 1) * 6:(i + 2) * 6] = bt.upper[i]
        full[(i + 1) * 6:(i + 2) * 6, i * 6:(i + 1) * 6] = bt.lower[i]
    assert np.array_equal(full, a.toarray())
    bad = a.tolil()
    bad[0, 29] = 1.0
    with pytest.raises(ValueError):
        block_partition(SparseOperator(bad.tocsr()), Mesh(p.nx, p.ny))


@pytest.mark.gpu
@pytest.mark.parametrize("name", RGF_CASES)
def test_rgf_matches_reference(cuda, name):
    from paper_1104_0623_b200 import Mesh, SparseOperator
    from paper_1104_0623_b200.rgf import rgf_batch

    g = load_golden(name)
    p = problem_from_golden(g)
    ops = [SparseOperator(p.a_csr(k)) for k in range(p.energies.size)]
    gr, gl, led = rgf_batch(Mesh(p.nx, p.ny), ops, SparseOperator(p.sigma_csr()))
    for k in range(p.energies.size):
        assert rel(gr[k], g["gr"][k]) < 1e-10
        assert rel(gl[k], g["gl"][k]) < 1e-10
    assert led["gr"].multiplications == golden_frac(g["W_gr"])
    assert led["gless"].multiplications == golden_frac(g["W_gl"])


@pytest.mark.gpu
def test_rgf_reference_signatures_and_find_agreement(cuda):
    """rgf_gr_diag / rgf_gless_diag with the reference's BlockTridiagonal inputs; RGF and
    FIND agree on cfg0 (40 x 40, dense contacts)."""
    from paper_1104_0623_b200 import FlopLedger, Mesh, SolverConfig, SparseOperator, solve
    from paper_1104_0623_b200.configs import config_problem
    from paper_1104_0623_b200.rgf import block_partition, rgf_gless_diag, rgf_gr_diag

    p = config_problem(0)
    mesh = Mesh(p.nx, p.ny)
    a, s = SparseOperator(p.a_csr(0)), SparseOperator(p.sigma_csr())
    led = FlopLedger()
    gr = rgf_gr_diag(block_partition(a, mesh), led)
    gl = rgf_gless_diag(block_partition(a, mesh), block_partition(s, mesh))
    assert led.multiplications > 0
    f = solve(mesh, a, s, SolverConfig())
    assert rel(gr, f.gr_diag) < 1e-10 and rel(gl, f.gless_diag) < 1e-10
