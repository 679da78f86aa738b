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
    """bench.py's cpu_baseline / --impl reference leg (oracle/cpu_baseline.py) on a tiny mesh: every
    elimination is in exactly one bucket, one member per bucket is timed."""
    from oracle.cpu_baseline import buckets_of, elimination_jobs, estimate_step
    from oracle.find_oracle import FindOracle
    from paper_1104_0623_b200.configs import build_problem

    p = build_problem(12, 10, [1.0], seed=2)
    o = FindOracle(p.nx, p.ny, p.a_csr(0))
    jobs = elimination_jobs(o)
    b = buckets_of(jobs)
    assert sum(len(v) for v in b.values()) == len(jobs)
    r = estimate_step(o, b, p.a_csr(0).tocsr(), p.sigma_csr().tocsr(), np.random.default_rng(0))
    assert r["seconds_per_energy"] > 0 and r["sampled_eliminations"] == len(b)
    # with every member below the cap the estimate is the timed part alone
    assert r["rate_part_seconds"] == 0.0


def test_cpu_baseline_rate_part():
    """Members above the cap are charged at the measured BLAS rate."""
    from oracle.cpu_baseline import buckets_of, elimination_jobs, estimate_step
    from oracle.find_oracle import FindOracle
    from paper_1104_0623_b200.configs import build_problem

    p = build_problem(12, 10, [1.0], seed=2)
    o = FindOracle(p.nx, p.ny, p.a_csr(0))
    b = buckets_of(elimination_jobs(o))
    wmax = max(j[4] for v in b.values() for j in v)
    r = estimate_step(o, b, p.a_csr(0).tocsr(), p.sigma_csr().tocsr(), np.random.default_rng(0), cap=wmax / 2)
    assert r["rate_part_seconds"] > 0 and r["blas_rate_cmults_per_s"] > 0


def test_cpu_baseline_energy_parallel_runs():
    """The energy-parallel CPU baseline (forked processes, one BLAS thread each) on a tiny mesh."""
    from oracle.cpu_baseline import energy_parallel
    from paper_1104_0623_b200.configs import build_problem

    p = build_problem(12, 10, [1.0, 2.0], seed=2)
    r = energy_parallel(0, steps=2, warmup=1, workers=2, problem=p)
    assert r["workers"] == 2 and len(r["steps"]) == 2
    for st in r["steps"]:
        assert st["rate"] > 0 and st["sampled"] > 0
        assert abs(st["rate"] - 2.0 / st["seconds_per_energy"]) < 0.5 * st["rate"]
