"""Synthetic inputs for the five BASELINE.json configurations.

One canonical, seeded generator shared by the GPU path, the oracle and the
bench: node (ix, iy) -> ix + Nx*iy; 5- or 9-point tight-binding H; dense
Nx x Nx contact self-energies on rows iy=0 (L) and iy=Ny-1 (R);
Sigma^< = i*Gamma_L; A(E) = (E + i*eta) I - H - Sigma_L - Sigma_R.

There is no public dataset behind these configs: BASELINE.json defines them
synthetically, and this recipe fixes the seed and order of
draws so every consumer sees identical arrays.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.sparse as sp

ETA = 1e-6


@dataclass(frozen=True)
class MeshConfig:
    index: int
    nx: int
    ny: int
    stencil: int
    vamp: float
    energies: tuple

    @property
    def n(self) -> int:
        return self.nx * self.ny

    @property
    def n_energies(self) -> int:
        return len(self.energies)


def _lin(n):
    return tuple(float(x) for x in np.linspace(0.5, 3.5, n))


CONFIGS = {
    0: MeshConfig(0, 40, 40, 5, 0.5, (1.0,)),
    1: MeshConfig(1, 130, 130, 5, 0.5, _lin(16)),
    2: MeshConfig(2, 256, 256, 9, 0.5, _lin(64)),
    3: MeshConfig(3, 256, 1024, 5, 1.0, _lin(32)),
    4: MeshConfig(4, 1024, 1024, 5, 0.5, _lin(8)),
}


@dataclass
class DeviceProblem:
    """CSR pattern shared by every energy; values per energy.

    ``pattern`` is the CSR (indptr, indices) of A (sorted indices, explicit
    zeros kept).  ``h_vals`` holds -H - Sigma_L - Sigma_R on that pattern,
    ``diag_pos`` the CSR slots of the diagonal, so A(E) values are
    ``h_vals + (E + i*eta)`` on ``diag_pos``.  ``s_vals`` is Sigma^< on A's
    pattern (zeros outside row iy=0).
    """

    nx: int
    ny: int
    indptr: np.ndarray
    indices: np.ndarray
    h_vals: np.ndarray
    diag_pos: np.ndarray
    s_vals: np.ndarray
    energies: np.ndarray

    @property
    def n(self):
        return self.nx * self.ny

    @property
    def nnz(self):
        return self.indices.size

    def a_vals(self, k: int) -> np.ndarray:
        v = self.h_vals.copy()
        v[self.diag_pos] += self.energies[k] + 1j * ETA
        return v

    def a_vals_all(self) -> np.ndarray:
        out = np.repeat(self.h_vals[None, :], self.energies.size, axis=0)
        out[:, self.diag_pos] += (self.energies + 1j * ETA)[:, None]
        return out

    def a_csr(self, k: int) -> sp.csr_matrix:
        return sp.csr_matrix((self.a_vals(k), self.indices, self.indptr), shape=(self.n, self.n))

    def sigma_csr(self) -> sp.csr_matrix:
        return sp.csr_matrix((self.s_vals, self.indices, self.indptr), shape=(self.n, self.n))


def build_problem(nx, ny, energies, seed=0, stencil=5, vamp=0.5) -> DeviceProblem:
    """BASELINE.md §3 steps 1-4 (draw order: V, then C_L, then C_R)."""
    rng = np.random.default_rng(seed)
    n = nx * ny
    v = rng.uniform(-vamp, vamp, n)
    ids = np.arange(n, dtype=np.int64).reshape(ny, nx)
    rows, cols, vals = [], [], []

    def hop(a, b, t):
        rows.extend([a, b])
        cols.extend([b, a])
        vals.extend([np.full(a.size, -t, complex), np.full(a.size, -t, complex)])

    hop(ids[:, :-1].ravel(), ids[:, 1:].ravel(), 1.0)
    hop(ids[:-1, :].ravel(), ids[1:, :].ravel(), 1.0)
    if stencil == 9:
        onsite = 5.0 + v
        hop(ids[:-1, :-1].ravel(), ids[1:, 1:].ravel(), 0.25)
        hop(ids[:-1, 1:].ravel(), ids[1:, :-1].ravel(), 0.25)
    elif stencil == 5:
        onsite = 4.0 + v
    else:
        raise ValueError("stencil must be 5 or 9")

    def contact():
        c = (rng.standard_normal((nx, nx)) + 1j * rng.standard_normal((nx, nx))) / np.sqrt(2.0)
        return -0.5j * (c @ c.conj().T) / nx

    sig_l, sig_r = contact(), contact()
    gam_l = 1j * (sig_l - sig_l.conj().T)
    sless = 1j * gam_l  # f_L = 1, f_R = 0
    lrow, rrow = ids[0, :], ids[ny - 1, :]

    def dense(block, nodes):
        rr, cc = np.meshgrid(nodes, nodes, indexing="ij")
        return rr.ravel(), cc.ravel(), block.ravel()

    h_r = np.concatenate([np.arange(n)] + rows)
    h_c = np.concatenate([np.arange(n)] + cols)
    h_v = np.concatenate([onsite.astype(complex)] + vals)
    lr, lc, lv = dense(sig_l, lrow)
    rr_, rc, rv = dense(sig_r, rrow)
    # -H - Sigma_L - Sigma_R (duplicates summed by scipy)
    m = sp.coo_matrix(
        (np.concatenate([-h_v, -lv, -rv]), (np.concatenate([h_r, lr, rr_]), np.concatenate([h_c, lc, rc]))),
        shape=(n, n),
    ).tocsr()
    m.sum_duplicates()
    m.sort_indices()
    sl_r, sl_c, sl_v = dense(sless, lrow)
    # Sigma^< on A's pattern
    for_rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(m.indptr))
    keys = for_rows * n + m.indices.astype(np.int64)  # ascending (sorted CSR)
    s_vals = np.zeros(m.nnz, dtype=complex)
    skeys = sl_r.astype(np.int64) * n + sl_c.astype(np.int64)
    pos = np.searchsorted(keys, skeys)
    if np.any(pos >= keys.size) or np.any(keys[np.minimum(pos, keys.size - 1)] != skeys):
        raise RuntimeError("Sigma^< pattern is not contained in A's pattern")
    np.add.at(s_vals, pos, sl_v)
    diag_pos = np.empty(n, dtype=np.int64)
    dmask = for_rows == m.indices
    diag_pos[for_rows[dmask]] = np.nonzero(dmask)[0]
    return DeviceProblem(nx, ny, m.indptr.astype(np.int64), m.indices.astype(np.int64), m.data.copy(),
                         diag_pos, s_vals, np.asarray(energies, float))


def config_problem(index: int, n_energies: int | None = None) -> DeviceProblem:
    cfg = CONFIGS[index]
    energies = np.asarray(cfg.energies if n_energies is None else cfg.energies[:n_energies])
    return build_problem(cfg.nx, cfg.ny, energies, seed=index, stencil=cfg.stencil, vamp=cfg.vamp)
