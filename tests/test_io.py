"""Data formats either side of the solve: Matrix Market (operators.py:222-244) and the
CSV exports (solver.py:709-734), pinned byte-for-byte against files the reference wrote
(tests/golden/make_golden.py io_cases)."""

import numpy as np
import pytest

from conftest import GOLDEN, load_golden


def _problem():
    from paper_1104_0623_b200.configs import build_problem

    return build_problem(6, 5, [1.2], seed=41, stencil=5)


@pytest.mark.parametrize("with_mesh", [True, False])
def test_matrix_market_write_matches_reference_bytes(tmp_path, with_mesh):
    from paper_1104_0623_b200 import Mesh, SparseOperator, write_matrix_market

    p = _problem()
    out = tmp_path / "a.mtx"
    write_matrix_market(out, SparseOperator(p.a_csr(0)), Mesh(p.nx, p.ny) if with_mesh else None)
    want = (GOLDEN / ("io_a_mesh.mtx" if with_mesh else "io_a_plain.mtx")).read_bytes()
    assert out.read_bytes() == want


@pytest.mark.parametrize("name,dims", [("io_a_mesh.mtx", (6, 5)), ("io_a_plain.mtx", None)])
def test_matrix_market_read_reference_file(name, dims):
    from paper_1104_0623_b200 import read_matrix_market

    op, got = read_matrix_market(GOLDEN / name)
    assert got == dims
    p = _problem()
    assert (op.matrix != p.a_csr(0)).nnz == 0


def test_csv_format_matches_reference_bytes():
    """The reference's own result values through our writers give the reference's bytes."""
    from paper_1104_0623_b200 import Mesh, diag_to_csv, offdiag_to_csv
    from paper_1104_0623_b200.ledger import FlopLedger
    from paper_1104_0623_b200.solver import SelectedInverse

    g = load_golden("io_csv")
    mesh = Mesh(int(g["nx"]), int(g["ny"]))
    off = {tuple(k): complex(v) for k, v in zip(g["off_keys"].tolist(), g["off_vals"])}
    r = SelectedInverse(g["gr"], g["gl"], off, FlopLedger())
    assert diag_to_csv(r, mesh) == str(g["diag_csv"])
    assert offdiag_to_csv(r) == str(g["offdiag_csv"])
    h = load_golden("io_csv_nogless")
    r2 = SelectedInverse(h["gr"], None, None, FlopLedger())
    assert diag_to_csv(r2, mesh) == str(h["diag_csv"])
    assert offdiag_to_csv(r2) == str(h["offdiag_csv"])


@pytest.mark.gpu
def test_csv_bytes_deterministic_and_batch_rows(cuda):
    """test_acceptance.py:392-402: identical CSV bytes across runs; the batch writer's row
    for one energy equals the single-solve writer's text."""
    from paper_1104_0623_b200 import (Mesh, SolverConfig, SparseOperator, diag_to_csv, offdiag_to_csv, solve,
                                      solve_batch)

    p = _problem()
    mesh = Mesh(p.nx, p.ny)
    a, s = SparseOperator(p.a_csr(0)), SparseOperator(p.sigma_csr())
    cfg = SolverConfig(compute_offdiag=True)
    r1, r2 = solve(mesh, a, s, cfg), solve(mesh, a, s, cfg)
    assert diag_to_csv(r1, mesh) == diag_to_csv(r2, mesh)
    assert offdiag_to_csv(r1) == offdiag_to_csv(r2)
    assert offdiag_to_csv(r1, gless=True) == offdiag_to_csv(r2, gless=True)
    rb = solve_batch(mesh, [a], s, cfg)
    assert diag_to_csv(rb, mesh, energy=0) == diag_to_csv(r1, mesh)
    assert offdiag_to_csv(rb, energy=0) == offdiag_to_csv(r1)
    assert offdiag_to_csv(rb, energy=0, gless=True) == offdiag_to_csv(r1, gless=True)
    g = load_golden("io_csv")
    assert np.max(np.abs(r1.gr_diag - g["gr"])) < 1e-10 * np.max(np.abs(g["gr"]))
