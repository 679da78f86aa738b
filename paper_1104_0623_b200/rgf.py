"""Block-tridiagonal recursive Green's function (RGF) on the GPU — the reference's
crossover baseline (find_selinv/rgf.py:1-208).

The operator is blocked by mesh rows (line y = nodes y*nx .. y*nx+nx-1), which makes it
block tridiagonal: D_i = A(line_i, line_i), E_i = A(line_i, line_{i+1}),
F_i = A(line_{i+1}, line_i).  The recurrences are those of the reference:

    g_0 = D_0^-1,  g_i = (D_i - F_{i-1} g_{i-1} E_{i-1})^-1                  (rgf.py:108-115)
    G_{N-1} = g_{N-1},  G_i = g_i + g_i E_i G_{i+1} F_i g_i                    (rgf.py:121-136)
    G^<: right-connected g^R, left/right-connected scattering blocks and
         G_ii R_i G_ii^H with R_i = S^L_i + S^R_i - S_ii                       (rgf.py:139-208)

Every step is batched over all energy points and runs on the library's own kernels
through the C ABI (include/find_b200.h): the inverses are find_dense_inverse (one blocked
elimination of [[A, I], [I, 0]] per matrix on the FIND panel / TRSM / DMMA kernels), the
products find_zgemm_batched (DMMA tiles, the subtraction / addition of the recurrences
folded into the accumulator); torch only holds the buffers and does the diagonal
scalings and element-wise sums.  The ledger follows the reference's charging rules
(rgf.py:89-107: inverse c^3, products skipped when the coupling block is diagonal).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

from .errors import NativeLibraryError, SingularPivotError
from .ledger import FlopLedger


@dataclass
class BlockTridiagonal:
    """rgf.py:28-40: line blocks D_i, E_i = A(line_i, line_{i+1}), F_i = A(line_{i+1}, line_i)."""

    diag: list
    upper: list
    lower: list
    lines: list

    @property
    def num_blocks(self) -> int:
        return len(self.diag)


def _check_tridiagonal(m: sp.csr_matrix, nx: int):
    c = m.tocoo()
    if np.any(np.abs(c.row // nx - c.col // nx) > 1):
        raise ValueError("operator pattern is not block tridiagonal over mesh lines")


def block_partition(op, mesh) -> BlockTridiagonal:
    """rgf.py:43-61 (host numpy blocks; same validation and error)."""
    if op.n != mesh.n:
        raise ValueError("operator size does not match the mesh")
    m = op.matrix.tocsr()
    _check_tridiagonal(m, mesh.nx)
    nx, ny = mesh.nx, mesh.ny
    lines = [np.arange(y * nx, (y + 1) * nx, dtype=np.int64) for y in range(ny)]
    blk = lambda r, c: m[r * nx:(r + 1) * nx, c * nx:(c + 1) * nx].toarray().astype(np.complex128)
    return BlockTridiagonal([blk(y, y) for y in range(ny)], [blk(y, y + 1) for y in range(ny - 1)],
                            [blk(y + 1, y) for y in range(ny - 1)], lines)


def _device():
    import torch

    if not torch.cuda.is_available():
        raise NativeLibraryError("the RGF path needs a CUDA device (there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


class _Lines:
    """Dense line blocks of a batch of CSR matrices sharing one pattern, built on the device one line at
    a time (D(i) / E(i) / F(i): [nE, nx, nx]); holding all 3 ny blocks at once is 48 GB per energy point
    at 1024 x 1024.  ediag / fdiag: the coupling blocks with no nonzero off their diagonal (rgf.py:75-81)."""

    def __init__(self, mats, nx: int, ny: int, dev):
        import torch

        self.nx, self.ny, self.dev, self.ne = nx, ny, dev, len(mats)
        m0 = mats[0].tocoo()
        r, c = m0.row.astype(np.int64), m0.col.astype(np.int64)
        ly, lc = r // nx, c // nx
        vals = np.stack([np.asarray(_coo_on(m, m0), np.complex128) for m in mats])
        self.vals = torch.from_numpy(vals).to(dev)
        local = (r % nx) * nx + c % nx
        offd = (r % nx) != (c % nx)
        self.idx, self.pos, self.off = {}, {}, {}
        nz_off = {}
        for kind, sel, line, nl in (("D", ly == lc, ly, ny), ("E", lc == ly + 1, ly, ny - 1), ("F", ly == lc + 1, lc, ny - 1)):
            where = np.nonzero(sel)[0]
            order = np.argsort(line[where], kind="stable")
            where = where[order]
            self.pos[kind] = torch.from_numpy(where).to(dev)
            self.idx[kind] = torch.from_numpy(local[where]).to(dev)
            self.off[kind] = np.searchsorted(line[where], np.arange(max(nl, 0) + 1))
            flag = np.zeros(max(nl, 0), bool)  # lines with a nonzero off-diagonal entry in some energy point
            hot = where[offd[where] & np.any(vals[:, where] != 0, axis=0)]
            flag[line[hot]] = True
            nz_off[kind] = flag
        self.ediag = [not bool(x) for x in nz_off["E"]]
        self.fdiag = [not bool(x) for x in nz_off["F"]]

    def _block(self, kind: str, i: int):
        import torch

        out = torch.zeros((self.ne, self.nx * self.nx), dtype=torch.complex128, device=self.dev)
        a, b = int(self.off[kind][i]), int(self.off[kind][i + 1])
        if b > a:
            out[:, self.idx[kind][a:b]] = self.vals[:, self.pos[kind][a:b]]  # (row, col) unique
        return out.view(self.ne, self.nx, self.nx)

    def D(self, i: int):
        return self._block("D", i)

    def E(self, i: int):
        return self._block("E", i)

    def F(self, i: int):
        return self._block("F", i)


def _coo_on(m, m0) -> np.ndarray:
    """Values of m on m0's COO pattern (m must share the pattern)."""
    m = m.tocsr()
    if m.nnz == m0.nnz:
        cm = m.tocoo()
        if np.array_equal(cm.row, m0.row) and np.array_equal(cm.col, m0.col):
            return cm.data
    return np.asarray(m[m0.row, m0.col]).ravel()


class _Dense:
    """The C-ABI dense primitives on torch buffers: batched inverse (one handle per (n, batch),
    cached) and strided-batched GEMM, both asynchronous on torch's current stream."""

    _handles: dict = {}

    def __init__(self, n: int, batch: int, dev):
        import ctypes as C
        import torch

        from . import _native

        self.L = _native.lib()
        self.C = C
        self.n, self.batch, self.dev = n, batch, dev
        key = (n, batch, dev.index)
        if key not in _Dense._handles:
            if len(_Dense._handles) >= 4:  # a few (n, batch) shapes at most: free the oldest workspace
                old = next(iter(_Dense._handles))
                self.L.find_dense_destroy(_Dense._handles.pop(old))
            h = C.c_void_p()
            st = _native.FindStatus()
            rc = self.L.find_dense_create(n, batch, C.byref(h), C.byref(st))
            if rc != 0:
                raise NativeLibraryError(f"find_dense_create failed: {st.text}")
            _Dense._handles[key] = h
        self.h = _Dense._handles[key]
        self.stream = C.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
        self._native = _native

    def inv(self, X, line: int, infos: list):
        """Batched inverse; the status words are collected and checked once per sweep
        (no host synchronisation per line)."""
        import torch

        X = X.contiguous()
        out = torch.empty_like(X)
        word = torch.empty(1, dtype=torch.int64, device=self.dev)
        st = self._native.FindStatus()
        rc = self.L.find_dense_inverse(self.h, X.data_ptr(), out.data_ptr(), word.data_ptr(), self.stream,
                                       self.C.byref(st))
        if rc != 0:
            raise NativeLibraryError(f"find_dense_inverse failed: {st.text}")
        infos.append((line, word))
        return out

    def mm(self, A, B, acc=None, mode: int = 0, bh: bool = False):
        """A @ B (mode 0), acc + A @ B (+1) or acc - A @ B (-1) per energy point; bh: B is used as its
        conjugate transpose.  A / B / acc: [nE or 1, n, n] complex128 on the device (a leading 1 broadcasts)."""
        import torch

        A, B = A.contiguous(), B.contiguous()
        n = self.n
        ne = max(A.shape[0], B.shape[0], acc.shape[0] if acc is not None else 1)
        out = torch.empty((ne, n, n), dtype=torch.complex128, device=self.dev)
        if acc is not None:
            out.copy_(acc)  # broadcasts a leading 1
        st = self._native.FindStatus()
        sa = 0 if A.shape[0] == 1 and ne > 1 else n * n
        sb = 0 if B.shape[0] == 1 and ne > 1 else n * n
        rc = self.L.find_zgemm_batched(ne, n, n, n, A.data_ptr(), n, sa, B.data_ptr(), n, sb, 1 if bh else 0,
                                       out.data_ptr(), n, n * n, mode if acc is not None else 0, self.stream,
                                       self.C.byref(st))
        if rc != 0:
            raise NativeLibraryError(f"find_zgemm_batched failed: {st.text}")
        return out


def _check_infos(infos: list):
    import torch

    if not infos:
        return
    bad = torch.cat([w for _, w in infos]).ne(-1).nonzero()
    if bad.numel():
        raise SingularPivotError(f"singular recurrence block at line {infos[int(bad[0, 0])][0]}")
    infos.clear()


def _sandwich(dn, L, Mid, R, ldiag: bool, rdiag: bool, acc=None, mode: int = 0):
    """L @ Mid @ R with diagonal factors applied as scalings (rgf.py:92-105); with acc / mode the
    result is added to (+1) or subtracted from (-1) acc inside the last product."""
    t = Mid
    t = t * L.diagonal(dim1=-2, dim2=-1).unsqueeze(-1) if ldiag else dn.mm(L, t)
    if rdiag:
        t = t * R.diagonal(dim1=-2, dim2=-1).unsqueeze(-2)
        return t if acc is None else (acc + t if mode > 0 else acc - t)
    return dn.mm(t, R, acc, mode)


def rgf_batch(mesh, a_list, sigma=None, compute_gless: bool = True):
    """diag(G^r) [nE, n] and, if requested, diag(G^<) [nE, n] of every operator in a_list
    (shared pattern, block tridiagonal over mesh lines) by the RGF recurrences, batched
    over the energy points on the device.  Returns (gr, gl, ledgers) with the per-energy
    reference ledgers of rgf_gr_diag (ledgers["gr"]) and rgf_gless_diag (ledgers["gless"])."""
    import torch

    dev = _device()
    nx, ny = mesh.nx, mesh.ny
    mats = [a.matrix.tocsr() for a in a_list]
    for m in mats[:1]:
        if m.shape[0] != mesh.n:
            raise ValueError("operator size does not match the mesh")
        _check_tridiagonal(m, nx)
    led = FlopLedger()  # forward + backward: rgf_gr_diag's charges
    infos: list = []
    dn = _Dense(nx, len(mats), dev)
    A = _Lines(mats, nx, ny, dev)
    ediag, fdiag = A.ediag, A.fdiag
    c3 = nx ** 3

    def charge_sandwich(ld, rd):
        if not ld:
            led.add("rgf", c3)
        if not rd:
            led.add("rgf", c3)

    # forward: left-connected g_i (rgf.py:108-115)
    gl_blk = [None] * ny
    gl_blk[0] = dn.inv(A.D(0), 0, infos)
    led.add("rgf", c3)
    for i in range(1, ny):
        gl_blk[i] = dn.inv(_sandwich(dn, A.F(i - 1), gl_blk[i - 1], A.E(i - 1), fdiag[i - 1], ediag[i - 1],
                                     A.D(i), -1), i, infos)
        charge_sandwich(fdiag[i - 1], ediag[i - 1])
        led.add("rgf", c3)
    led_forward = FlopLedger(led.multiplications, dict(led.by_kernel))
    # backward: diagonal blocks of G (rgf.py:121-136)
    gr = torch.empty((len(mats), mesh.n), dtype=torch.complex128, device=dev)
    g_full = gl_blk[ny - 1]
    gr[:, (ny - 1) * nx:] = g_full.diagonal(dim1=-2, dim2=-1)
    for i in range(ny - 2, -1, -1):
        t = _sandwich(dn, A.E(i), g_full, A.F(i), ediag[i], fdiag[i])
        charge_sandwich(ediag[i], fdiag[i])
        g_full = dn.mm(dn.mm(gl_blk[i], t), gl_blk[i], gl_blk[i], +1)
        led.add("rgf", 2 * c3)
        gr[:, i * nx:(i + 1) * nx] = g_full.diagonal(dim1=-2, dim2=-1)
    _check_infos(infos)
    led_gr = led
    led = FlopLedger(led_forward.multiplications, dict(led_forward.by_kernel))  # rgf_gless_diag's charges
    if not compute_gless:
        return gr.cpu().numpy(), None, {"gr": led_gr, "gless": None}
    if sigma is None:
        raise ValueError("compute_gless requires a scattering matrix")
    sm = sigma.matrix.tocsr()
    _check_tridiagonal(sm, nx)
    S = _Lines([sm], nx, ny, dev)  # Sigma^< is energy independent
    sc = sm.tocoo()
    up_nz = np.zeros(max(ny - 1, 0), bool)  # Sigma coupling blocks with a nonzero entry (host, no sync)
    lo_nz = np.zeros(max(ny - 1, 0), bool)
    nzm = sc.data != 0
    up_nz[(sc.row // nx)[nzm & (sc.col // nx == sc.row // nx + 1)]] = True
    lo_nz[(sc.col // nx)[nzm & (sc.row // nx == sc.col // nx + 1)]] = True
    # right-connected g^R (rgf.py:164-168; its ledger repeats the forward one)
    gr_blk = [None] * ny
    gr_blk[ny - 1] = dn.inv(A.D(ny - 1), ny - 1, infos)
    led.add("rgf", c3)
    for i in range(ny - 2, -1, -1):
        gr_blk[i] = dn.inv(_sandwich(dn, A.E(i), gr_blk[i + 1], A.F(i), ediag[i], fdiag[i], A.D(i), -1), i, infos)
        charge_sandwich(ediag[i], fdiag[i])
        led.add("rgf", c3)

    def connected(g_conn, reverse):  # rgf.py:139-178
        s_conn = [None] * ny
        order = range(ny - 1, -1, -1) if reverse else range(ny)
        prev = None
        for i in order:
            if prev is None:
                s_conn[i] = S.D(i)
            else:
                if reverse:
                    coup, cdiag = A.E(i), ediag[i]
                    nz_sb, nz_bs = lo_nz[i], up_nz[i]
                    sig_sb, sig_bs = (S.F(i) if nz_sb else None), (S.E(i) if nz_bs else None)
                else:
                    coup, cdiag = A.F(i - 1), fdiag[i - 1]
                    nz_sb, nz_bs = up_nz[i - 1], lo_nz[i - 1]
                    sig_sb, sig_bs = (S.E(i - 1) if nz_sb else None), (S.F(i - 1) if nz_bs else None)
                if cdiag:
                    l_fac = coup.diagonal(dim1=-2, dim2=-1).unsqueeze(-1) * g_conn[prev]
                else:
                    l_fac = dn.mm(coup, g_conn[prev])
                    led.add("rgf", c3)
                term = dn.mm(dn.mm(l_fac, s_conn[prev]), l_fac, S.D(i), +1, bh=True)
                led.add("rgf", 2 * c3)
                if nz_sb:
                    term = dn.mm(l_fac, sig_sb, term, -1)
                if nz_bs:
                    term = dn.mm(sig_bs, l_fac, term, -1, bh=True)
                s_conn[i] = term
            prev = i
        return s_conn

    s_left = connected(gl_blk, False)
    s_right = connected(gr_blk, True)
    gless = torch.empty_like(gr)
    for i in range(ny):  # rgf.py:193-207
        u = A.D(i)
        if i > 0:
            u = _sandwich(dn, A.F(i - 1), gl_blk[i - 1], A.E(i - 1), fdiag[i - 1], ediag[i - 1], u, -1)
            charge_sandwich(fdiag[i - 1], ediag[i - 1])
        if i + 1 < ny:
            u = _sandwich(dn, A.E(i), gr_blk[i + 1], A.F(i), ediag[i], fdiag[i], u, -1)
            charge_sandwich(ediag[i], fdiag[i])
        r_i = s_left[i] + s_right[i] - S.D(i)
        s_left[i] = s_right[i] = None  # (release the line's connected blocks)
        g_ii = dn.inv(u, i, infos)
        led.add("rgf", c3)
        gless[:, i * nx:(i + 1) * nx] = dn.mm(dn.mm(g_ii, r_i), g_ii, bh=True).diagonal(dim1=-2, dim2=-1)
        led.add("rgf", 2 * c3)
    _check_infos(infos)
    return gr.cpu().numpy(), gless.cpu().numpy(), {"gr": led_gr, "gless": led}


def rgf_gr_diag(bt: BlockTridiagonal, ledger: FlopLedger | None = None) -> np.ndarray:
    """rgf.py:118-136 on the device, for one operator given as line blocks."""
    gr, _, led = _rgf_from_blocks(bt, None, False)
    if ledger is not None:
        ledger.merge(led["gr"])
    return gr


def rgf_gless_diag(bt: BlockTridiagonal, sigma_bt: BlockTridiagonal, ledger: FlopLedger | None = None) -> np.ndarray:
    """rgf.py:181-208 on the device, for one operator and scattering matrix given as line blocks."""
    _, gl, led = _rgf_from_blocks(bt, sigma_bt, True)
    if ledger is not None:
        ledger.merge(led["gless"])
    return gl


def _rgf_from_blocks(bt, sigma_bt, gless):
    from .mesh import Mesh
    from .operators import SparseOperator

    nx = bt.lines[0].size
    ny = bt.num_blocks
    n = nx * ny

    def assemble(b):
        m = sp.lil_matrix((n, n), dtype=np.complex128)
        for i in range(ny):
            m[i * nx:(i + 1) * nx, i * nx:(i + 1) * nx] = b.diag[i]
            if i + 1 < ny:
                m[i * nx:(i + 1) * nx, (i + 1) * nx:(i + 2) * nx] = b.upper[i]
                m[(i + 1) * nx:(i + 2) * nx, i * nx:(i + 1) * nx] = b.lower[i]
        return SparseOperator(m.tocsr())

    a = assemble(bt)
    s = assemble(sigma_bt) if sigma_bt is not None else None
    gr, gl, led = rgf_batch(Mesh(nx, ny), [a], s, gless)
    return gr[0], (gl[0] if gl is not None else None), led
