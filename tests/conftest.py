import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_golden(name):
    return np.load(GOLDEN / f"{name}.npz", allow_pickle=True)


def golden_frac(arr):
    from fractions import Fraction

    return Fraction(int(arr[0]), int(arr[1]))


def problem_from_golden(g):
    from paper_1104_0623_b200.configs import DeviceProblem

    return DeviceProblem(int(g["nx"]), int(g["ny"]), g["indptr"], g["indices"], g["h_vals"], g["diag_pos"],
                         g["s_vals"], g["energies"])


def stencil_ops(g):
    """(mesh, A, Sigma) of a golden stencil case (reference conftest.py:11-78 generators)."""
    import scipy.sparse as sp

    from paper_1104_0623_b200 import Mesh, SparseOperator

    nx, ny = int(g["nx"]), int(g["ny"])
    n = nx * ny
    a = SparseOperator(sp.csr_matrix((g["a_data"], g["a_indices"], g["a_indptr"]), shape=(n, n)))
    s = SparseOperator(sp.csr_matrix((g["s_data"], g["s_indices"], g["s_indptr"]), shape=(n, n)))
    return Mesh(nx, ny), a, s


def stencil_operator(nx, ny, seed, kind="general"):
    """Seeded diagonally dominant operator on the 5-point pattern (restates reference conftest.py:11-51)."""
    from paper_1104_0623_b200 import SparseOperator, build_mesh

    mesh = build_mesh(nx, ny)
    rng = np.random.default_rng(seed)
    adj = mesh.adjacency().tocoo()
    mask = adj.row < adj.col
    rows, cols = adj.row[mask], adj.col[mask]
    m = rows.size
    degree = np.asarray(mesh.adjacency().sum(axis=1)).ravel()
    hop = rng.standard_normal(m) + 1j * rng.standard_normal(m)
    if kind == "general":
        back = rng.standard_normal(m) + 1j * rng.standard_normal(m)
        diag = degree * 1.6 + 1.0 + rng.random(mesh.n) + 1j * (1.0 + rng.random(mesh.n))
    elif kind == "hermitian_pd":
        back = hop.conj()
        diag = degree * (np.abs(hop).max() + 0.3) + 1.0 + rng.random(mesh.n)
    else:
        raise ValueError(kind)
    ids = np.arange(mesh.n)
    op = SparseOperator.from_coo(mesh.n, np.concatenate([ids, rows, cols]), np.concatenate([ids, cols, rows]),
                                 np.concatenate([diag.astype(complex), hop, back]))
    return mesh, op


def stencil_sigma(mesh, seed, mode="diagonal"):
    from paper_1104_0623_b200 import SparseOperator

    rng = np.random.default_rng(seed)
    ids = np.arange(mesh.n)
    if mode == "diagonal":
        vals = rng.standard_normal(mesh.n) + 1j * rng.standard_normal(mesh.n)
        return SparseOperator.from_coo(mesh.n, ids, ids, vals.astype(complex))
    adj = mesh.adjacency().tocoo()
    mask = adj.row < adj.col
    rows, cols = adj.row[mask], adj.col[mask]
    hop = rng.standard_normal(rows.size) + 1j * rng.standard_normal(rows.size)
    back = rng.standard_normal(rows.size) + 1j * rng.standard_normal(rows.size)
    diag = rng.standard_normal(mesh.n) + 1j * rng.standard_normal(mesh.n)
    return SparseOperator.from_coo(mesh.n, np.concatenate([ids, rows, cols]), np.concatenate([ids, cols, rows]),
                                   np.concatenate([diag.astype(complex), hop, back]))


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)
