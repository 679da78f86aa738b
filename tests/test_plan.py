"""Native plan builder vs the reference's node sets and ledger (CPU only)."""

from fractions import Fraction

import numpy as np
import pytest

from conftest import golden_frac, load_golden, problem_from_golden, stencil_ops
from paper_1104_0623_b200.plan import Plan


@pytest.mark.parametrize("name", ["sets_c5_12x10", "sets_c9_9x14"])
@pytest.mark.parametrize("lm", [1, 2, 3])
def test_sets_match_reference(name, lm):
    g = load_golden(f"{name}_lm{lm}")
    plan = Plan(int(g["nx"]), int(g["ny"]), g["indptr"], g["indices"], lm)
    flat, offs = g["flat"], g["offs"]
    k = 0
    for label in g["labels"]:
        for which in range(5):
            ref = flat[offs[k]:offs[k + 1]]
            k += 1
            got = plan.cluster_set(int(label), which)
            assert np.array_equal(got, ref), (label, which)
    assert plan.info["n_clusters"] == len(g["labels"])


@pytest.mark.parametrize("name", ["cfg0", "c5_16x12", "c9_20x20", "c5_8x30"])
def test_work_matches_reference_ledger(name):
    g = load_golden(name)
    p = problem_from_golden(g)
    plan = Plan(p.nx, p.ny, p.indptr, p.indices)
    W = golden_frac(g["W"])
    assert plan.native_work(0) == W
    assert plan.ledger("naive").multiplications == W
    for kid, kern in enumerate(("parallel_inverse", "sequential_inverse", "block_lu", "naive_lu"), start=1):
        key = f"W_{kern}"
        if key in g.files:
            ref = golden_frac(g[key])
            assert plan.ledger(kern).multiplications == ref, kern
            assert plan.native_work(kid) == ref, kern


@pytest.mark.parametrize("name", ["c5_16x12", "c9_20x20", "c5_8x30"])
def test_exception_stats_match_reference(name):
    from paper_1104_0623_b200.solver import _stats

    g = load_golden(name)
    p = problem_from_golden(g)
    plan = Plan(p.nx, p.ny, p.indptr, p.indices)
    st = _stats(plan, p.a_vals(0))
    assert st["upward_exception_entries"] == int(g["stats_up_block_lu"])
    assert st["downward_exception_entries"] == int(g["stats_down_block_lu"])


@pytest.mark.parametrize("name", ["stencil_6x4", "stencil_3x5", "stencil_8x8", "stencil_16x16"])
@pytest.mark.parametrize("lm", [1, 2, 3])
def test_work_stencil_leaf_max(name, lm):
    g = load_golden(name)
    mesh, a, s = stencil_ops(g)
    if f"W_{lm}" not in g.files:
        pytest.skip("no golden")
    plan = Plan(mesh.nx, mesh.ny, a.matrix.indptr, a.matrix.indices, lm)
    assert plan.ledger("naive").multiplications == golden_frac(g[f"W_{lm}"])


def test_baseline_work_table():
    """exact W per energy point for cfg1 (cfg0 is in test_work_matches_reference_ledger)."""
    from paper_1104_0623_b200.configs import config_problem

    p = config_problem(1, 1)
    plan = Plan(p.nx, p.ny, p.indptr, p.indices)
    assert plan.native_work(0) == Fraction(10293205246, 3)


def test_schedule_covers_every_node_once():
    from paper_1104_0623_b200.configs import build_problem

    p = build_problem(13, 9, [1.0], seed=3, stencil=9)
    plan = Plan(p.nx, p.ny, p.indptr, p.indices)
    fin = plan.kind == 3
    assert int(plan.b[fin].sum()) == p.n  # leaves partition the mesh
    assert int(plan.groups["count"].sum()) == plan.info["n_elims"]
    # upward groups first (deepest level first), then downward/final by level
    passes = plan.groups["pass"]
    assert np.all(np.diff((passes > 0).astype(int)) >= 0)


def test_invalid_pattern_rejected():
    with pytest.raises(ValueError):
        Plan(2, 2, np.array([0, 1, 2, 3, 5]), np.array([0, 1, 2, 3, 9]))
    with pytest.raises(ValueError):
        Plan(0, 2, np.array([0]), np.array([], np.int64))


def test_single_cluster_mesh_plan():
    ids = np.arange(4)
    plan = Plan(2, 2, np.arange(5), ids)
    assert plan.info["n_elims"] == 1 and plan.kind[0] == 3 and plan.b[0] == 4
