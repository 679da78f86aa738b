"""Pass-level drop-in API (paper_1104_0623_b200/passes.py; reference solver.py:256-484):
upward / downward blocks against the CPU oracle's restatement of the same passes, leaf
extractions against dense inversion."""

import numpy as np
import pytest

from conftest import ROOT  # noqa: F401


def _problem():
    from paper_1104_0623_b200 import Mesh, SparseOperator
    from paper_1104_0623_b200.configs import build_problem

    p = build_problem(10, 8, [1.3], seed=31, stencil=5)
    return p, Mesh(p.nx, p.ny), SparseOperator(p.a_csr(0)), SparseOperator(p.sigma_csr())


def _oracle_passes(p):
    """The oracle's upward dict {label: (U, R)} and downward dict {-label: (U, R)}
    (oracle/find_oracle.py FindOracle.solve, passes kept)."""
    from oracle.find_oracle import FindOracle, OLedger, extract

    a, sg = p.a_csr(0), p.sigma_csr()
    o = FindOracle(p.nx, p.ny, a)
    led = OLedger()
    empty = np.array([], np.int64)
    z = np.zeros((0, 0), np.complex128)
    pos = {}
    for c in o.bottom_up:
        if c.parent is None:
            continue
        if c.is_leaf:
            order = np.concatenate([c.private_inner, c.boundary])
            pos[c.label] = o._eliminate(a, sg, order, empty, extract(a, order, order), z, extract(sg, order, order),
                                        z, c.private_inner, c.label, True, led, 1e-12)
        else:
            i, j = c.children
            pos[c.label] = o._eliminate(a, sg, i.boundary, j.boundary, pos[i.label][0], pos[j.label][0],
                                        pos[i.label][1], pos[j.label][1], c.private_inner, c.label, True, led, 1e-12)
    neg = {-1: (z, z)}
    stack = [o.root]
    while stack:
        c = stack.pop()
        if c.parent is not None:
            pr = c.parent
            a0, a1 = pr.children
            sib = a1 if a0 is c else a0
            neg[-c.label] = o._eliminate(a, sg, o.comps[-pr.label][0], sib.boundary, neg[-pr.label][0],
                                         pos[sib.label][0], neg[-pr.label][1], pos[sib.label][1],
                                         o.comps[-c.label][1], -c.label, True, led, 1e-12)
        stack.extend(reversed(c.children))
    return o, pos, neg


@pytest.mark.gpu
def test_upward_and_downward_pass_blocks(cuda):
    from paper_1104_0623_b200 import FlopLedger, SolverConfig, build_cluster_tree, downward_pass, upward_pass

    p, mesh, a, s = _problem()
    tree = build_cluster_tree(mesh, 2)
    led = FlopLedger()
    up = upward_pass(tree, a, s, SolverConfig(), ledger=led)
    o, pos, neg = _oracle_passes(p)
    assert set(up) == set(pos)
    for label, (u, r) in pos.items():
        scale = max(np.abs(u).max(), 1.0)
        assert np.abs(up[label].u.values - u).max() <= 1e-12 * scale, label
        assert np.abs(up[label].r.values - r).max() <= 1e-12 * max(np.abs(r).max(), 1.0), label
        np.testing.assert_array_equal(up[label].u.row_labels, o.by_label[label].boundary)
    seen = []
    down = downward_pass(tree, a, s, up, SolverConfig(), ledger=led, leaf_callback=lambda c, d: seen.append(c.label))
    for label, (u, r) in neg.items():
        if label == -1:
            continue
        assert np.abs(down[label].u.values - u).max() <= 1e-11 * max(np.abs(u).max(), 1.0), label
        assert np.abs(down[label].r.values - r).max() <= 1e-11 * max(np.abs(r).max(), 1.0), label
    leaves = [c.label for c in o.by_label.values() if c.is_leaf]
    assert sorted(seen) == sorted(leaves) and len(seen) == len(leaves)
    assert led.multiplications > 0


@pytest.mark.gpu
def test_downward_pass_consumes_given_cluster_data(cuda):
    """Perturbing the upward data changes the complement blocks (the pass reads what it is given)."""
    from paper_1104_0623_b200 import SolverConfig, build_cluster_tree, downward_pass, upward_pass

    p, mesh, a, s = _problem()
    tree = build_cluster_tree(mesh, 2)
    up = upward_pass(tree, a, s, SolverConfig())
    d0 = downward_pass(tree, a, s, up, SolverConfig())
    k = max(up, key=lambda x: up[x].u.values.size)
    up[k].u.values[...] *= 1.5
    d1 = downward_pass(tree, a, s, up, SolverConfig())
    assert any(np.abs(d1[x].u.values - d0[x].u.values).max() > 1e-6 for x in d0 if d0[x].u.values.size)


@pytest.mark.gpu
def test_leaf_extractions_match_dense(cuda):
    from paper_1104_0623_b200 import (SolverConfig, build_cluster_tree, downward_pass, leaf_extract_gless,
                                      leaf_extract_gr, leaf_extract_offdiag, upward_pass)
    from paper_1104_0623_b200.mesh import annotated_tree
    from paper_1104_0623_b200.plan import plan_for

    p, mesh, a, s = _problem()
    tree = build_cluster_tree(mesh, 2)
    up = upward_pass(tree, a, s, SolverConfig())
    down = downward_pass(tree, a, s, up, SolverConfig())
    plan, _ = plan_for(p.nx, p.ny, p.indptr, p.indices)
    atree, comps = annotated_tree(plan)
    A = a.to_dense()
    G = np.linalg.inv(A)
    GL = G @ s.to_dense() @ G.conj().T
    checked = 0
    for leaf in atree.leaves[::7]:
        ring = comps[-leaf.label].boundary
        nodes = leaf.nodes
        g = leaf_extract_gr(leaf, a, down[-leaf.label], ring)
        assert np.abs(g.values - G[np.ix_(nodes, nodes)]).max() <= 1e-10 * np.abs(G).max()
        gl = leaf_extract_gless(leaf, a, s, down[-leaf.label], ring)
        assert np.abs(gl.values - GL[np.ix_(nodes, nodes)]).max() <= 1e-10 * np.abs(GL).max()
        off = leaf_extract_offdiag(leaf, a, down[-leaf.label], ring, g.values)
        for (u, v), val in off.items():
            assert abs(val - G[u, v]) <= 1e-10 * np.abs(G).max(), (u, v)
        checked += 1
    assert checked >= 3
