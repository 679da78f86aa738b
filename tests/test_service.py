"""The reference's service-handler tests (find_selinv tests/test_service.py:30-60) against the B200
handlers: Matrix Market text in, the GPU solve, JSON-like fields and CSV out."""

import numpy as np
import pytest

from conftest import stencil_operator


def dense_gr_diag(a):
    return np.diag(np.linalg.inv(a))


@pytest.fixture()
def mtx_pair(tmp_path):
    from paper_1104_0623_b200 import SparseOperator, write_matrix_market

    mesh, a = stencil_operator(6, 5, seed=11)
    rng = np.random.default_rng(5)
    c = rng.standard_normal((mesh.n, 3)) + 1j * rng.standard_normal((mesh.n, 3))
    import scipy.sparse as sp

    pat = (abs(a.matrix) > 0).astype(float)
    sigma = SparseOperator(sp.csr_matrix(pat.multiply(1j * (c @ c.conj().T))))
    ap, spth = tmp_path / "a.mtx", tmp_path / "s.mtx"
    write_matrix_market(ap, a, mesh)
    write_matrix_market(spth, sigma, mesh)
    return mesh, a, sigma, ap, spth


@pytest.mark.gpu
def test_handle_solve_matches_dense(cuda, mtx_pair):
    from paper_1104_0623_b200.service import SolveRequest, handle_solve

    mesh, a, sigma, ap, sp = mtx_pair
    resp = handle_solve(SolveRequest(matrix_mtx=ap.read_text(), sigma_mtx=sp.read_text(), kernel="block_lu"))
    got = np.array([complex(re, im) for re, im in resp.gr_diag])
    ref = dense_gr_diag(a.matrix.toarray())
    assert np.max(np.abs(got - ref) / np.abs(ref)) < 1e-10
    g = np.linalg.inv(a.matrix.toarray())
    gl_ref = np.diag(g @ sigma.matrix.toarray() @ g.conj().T)
    gl = np.array([complex(re, im) for re, im in resp.gless_diag])
    assert np.max(np.abs(gl - gl_ref)) / np.max(np.abs(gl_ref)) < 1e-10
    assert resp.nx == 6 and resp.ny == 5  # from the %%mesh header
    assert resp.diag_csv.startswith("node,x,y,")
    assert resp.flops > 0 and "block_lu" in " ".join(resp.flops_breakdown)


@pytest.mark.gpu
def test_handle_solve_requires_mesh_dims(cuda, tmp_path):
    from paper_1104_0623_b200 import write_matrix_market
    from paper_1104_0623_b200.service import SolveRequest, handle_solve

    mesh, a = stencil_operator(2, 2, seed=3)
    path = tmp_path / "a.mtx"
    write_matrix_market(path, a)  # no %%mesh header
    with pytest.raises(ValueError):
        handle_solve(SolveRequest(matrix_mtx=path.read_text(), compute_gless=False))
    resp = handle_solve(SolveRequest(matrix_mtx=path.read_text(), nx=2, ny=2, compute_gless=False))
    assert resp.nx == 2 and resp.gless_diag is None


@pytest.mark.gpu
def test_handle_solve_offdiag(cuda, mtx_pair):
    from paper_1104_0623_b200.service import SolveRequest, handle_solve

    mesh, a, sigma, ap, sp = mtx_pair
    resp = handle_solve(SolveRequest(matrix_mtx=ap.read_text(), sigma_mtx=sp.read_text(), compute_offdiag=True))
    g = np.linalg.inv(a.matrix.toarray())
    assert resp.offdiag and resp.offdiag_csv
    for ent in resp.offdiag[:20]:
        assert abs(complex(ent.re, ent.im) - g[ent.i, ent.j]) < 1e-10 * np.abs(g).max()


def test_handle_model_single_and_all():
    from paper_1104_0623_b200.service import ModelRequest, handle_health, handle_model

    resp = handle_model(ModelRequest(kernel="parallel_inverse", m=64, n=192))
    assert resp.entries[0].cost == pytest.approx(float(152 * 64**3 / 3))
    all_resp = handle_model(ModelRequest(s=8, b=8, m=4, n=4))
    assert len(all_resp.entries) > 10
    with pytest.raises(ValueError):
        handle_model(ModelRequest(kernel="parallel_inverse"))
    assert handle_health()["status"] == "ok"
