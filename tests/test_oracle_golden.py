"""Pin the CPU oracle (oracle/find_oracle.py) against the reference's own outputs."""

import numpy as np
import pytest

from conftest import golden_frac, load_golden, problem_from_golden, stencil_ops
from oracle.find_oracle import FindOracle, dense_gless_diag, dense_gr_diag, work_naive


@pytest.mark.parametrize("name", ["c5_16x12", "c9_20x20", "c5_8x30", "cfg0"])
def test_oracle_matches_reference_contacts(name):
    g = load_golden(name)
    p = problem_from_golden(g)
    o = FindOracle(p.nx, p.ny, p.a_csr(0))
    energies = range(p.energies.size) if name != "cfg0" else [0]
    for k in energies:
        r = o.solve(p.a_csr(k), p.sigma_csr())
        assert np.abs(r.gr_diag - g["gr"][k]).max() / np.abs(g["gr"][k]).max() < 1e-13
        assert np.abs(r.gless_diag - g["gl"][k]).max() / np.abs(g["gl"][k]).max() < 1e-13
        assert r.ledger.multiplications == golden_frac(g["W"])
    assert work_naive(o) == golden_frac(g["W"])


@pytest.mark.parametrize("name", ["stencil_6x4", "stencil_4x4", "stencil_3x5", "stencil_5x7", "stencil_8x8"])
@pytest.mark.parametrize("leaf_max", [1, 2, 3])
def test_oracle_matches_reference_stencil(name, leaf_max):
    g = load_golden(name)
    mesh, a, s = stencil_ops(g)
    o = FindOracle(mesh.nx, mesh.ny, a.matrix, leaf_max)
    r = o.solve(a.matrix, s.matrix)
    np.testing.assert_allclose(r.gr_diag, g[f"gr_{leaf_max}"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(r.gless_diag, g[f"gl_{leaf_max}"], rtol=1e-12, atol=1e-14)
    assert r.ledger.multiplications == golden_frac(g[f"W_{leaf_max}"])


def test_oracle_matches_dense_small():
    g = load_golden("stencil_6x4")
    mesh, a, s = stencil_ops(g)
    o = FindOracle(mesh.nx, mesh.ny, a.matrix)
    r = o.solve(a.matrix, s.matrix)
    assert np.max(np.abs(r.gr_diag - dense_gr_diag(a.to_dense())) / np.abs(g["dense_gr"])) < 1e-10
    assert np.max(np.abs(r.gless_diag - dense_gless_diag(a.to_dense(), s.to_dense())) / np.abs(g["dense_gl"])) < 1e-10


def test_cpu_baseline_estimator_runs():
    """bench.py's cpu_baseline / --impl reference leg (oracle/cpu_baseline.py) on a tiny mesh."""
    from oracle.cpu_baseline import estimate_seconds_per_energy
    from oracle.find_oracle import FindOracle
    from paper_1104_0623_b200.configs import build_problem

    p = build_problem(12, 10, [1.0], seed=2)
    o = FindOracle(p.nx, p.ny, p.a_csr(0))
    r = estimate_seconds_per_energy(o, p.a_csr(0), p.sigma_csr(), fraction=0.5, seed=0)
    assert r["seconds_per_energy"] > 0 and r["sampled_eliminations"] > 0


def test_cpu_baseline_energy_parallel_runs():
    """The energy-parallel CPU baseline (one process per core, one BLAS thread each) on a tiny mesh."""
    from oracle.cpu_baseline import parallel_energy_rate
    from paper_1104_0623_b200.configs import build_problem

    p = build_problem(12, 10, [1.0], seed=2)
    r = parallel_energy_rate(p.nx, p.ny, p.a_csr(0).tocsr(), p.sigma_csr().tocsr(), workers=2, fraction=0.5)
    assert r["workers"] == 2 and r["rate"] > 0 and r["sampled_eliminations"] > 0
    assert abs(r["rate"] - 2.0 / r["seconds_per_energy"]) < 0.5 * r["rate"]
