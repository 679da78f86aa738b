"""The dense batched primitives of the C ABI (find_dense_inverse, find_zgemm_batched: the
kernels under the GPU RGF path) against numpy, through ctypes."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rand(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


@pytest.mark.parametrize("n,batch", [(1, 2), (5, 3), (16, 2), (20, 3), (33, 2), (100, 2), (257, 2), (600, 1)])
def test_dense_inverse_matches_numpy(cuda, n, batch):
    """Every path of the elimination kernels (warp n2 <= 32, CTA-in-smem n2 <= 64, blocked panels above)."""
    import torch

    from paper_1104_0623_b200.rgf import _Dense

    rng = np.random.default_rng(n)
    a = _rand(rng, batch, n, n) + 0.5 * n ** 0.5 * np.eye(n)
    dev = torch.device("cuda", 0)
    dn = _Dense(n, batch, dev)
    infos = []
    out = dn.inv(torch.from_numpy(a).to(dev), 0, infos).cpu().numpy()
    ref = np.linalg.inv(a)
    assert np.max(np.abs(out - ref)) / np.max(np.abs(ref)) < 1e-11
    assert int(infos[0][1].item()) == -1


def test_dense_inverse_flags_a_singular_matrix(cuda):
    import torch

    from paper_1104_0623_b200.errors import SingularPivotError
    from paper_1104_0623_b200.rgf import _check_infos, _Dense

    a = np.zeros((2, 40, 40), np.complex128)
    a[0] = np.eye(40)
    a[1] = np.eye(40)
    a[1, 7, 7] = 0.0  # second matrix exactly singular
    dev = torch.device("cuda", 0)
    infos = []
    _Dense(40, 2, dev).inv(torch.from_numpy(a).to(dev), 11, infos)
    with pytest.raises(SingularPivotError, match="line 11"):
        _check_infos(infos)


@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (7, 5, 3), (64, 64, 16), (65, 130, 47), (200, 96, 257)])
@pytest.mark.parametrize("bh", [False, True])
@pytest.mark.parametrize("mode", [0, 1, -1])
def test_zgemm_batched_matches_numpy(cuda, m, n, k, bh, mode):
    import torch

    from paper_1104_0623_b200 import _native

    L = _native.lib()
    rng = np.random.default_rng(m * 1000 + n * 10 + k)
    batch = 3
    a = _rand(rng, batch, m, k)
    b = _rand(rng, 1, n, k) if bh else _rand(rng, 1, k, n)  # broadcast B over the batch
    c = _rand(rng, batch, m, n)
    dev = torch.device("cuda", 0)
    A, B, Cc = (torch.from_numpy(x).to(dev) for x in (a, b, c))
    st = _native.FindStatus()
    rc = L.find_zgemm_batched(batch, m, n, k, A.data_ptr(), k, m * k, B.data_ptr(), k if bh else n, 0, int(bh),
                              Cc.data_ptr(), n, m * n, mode, C.c_void_p(torch.cuda.current_stream().cuda_stream),
                              C.byref(st))
    assert rc == 0, st.text
    prod = a @ (np.conj(np.swapaxes(b, -1, -2)) if bh else b)
    ref = prod if mode == 0 else c + mode * prod
    assert np.max(np.abs(Cc.cpu().numpy() - ref)) / np.max(np.abs(ref)) < 1e-13
