"""Exact multiplication ledger and closed-form cost model.

Restates find_selinv/kernels.py:43-146 (FlopLedger, flop_model) and the
charging rules of solver.py:135-172, 388, 404-410, 664: counts are complex
multiplications only, exact rationals, charged per elimination from the
plan's (kind, s, b) table.  The GPU executes one arithmetic for every
kernel name; the ledger reports what the reference charges for the chosen
``SolverConfig.kernel`` (the paper's flop count).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np


@dataclass
class FlopLedger:
    """Counted multiplications, mergeable, with a per-kernel breakdown (kernels.py:48-71)."""

    multiplications: Fraction = Fraction(0)
    by_kernel: dict = field(default_factory=dict)

    def add(self, kernel: str, count) -> None:
        count = Fraction(count)
        self.multiplications += count
        self.by_kernel[kernel] = self.by_kernel.get(kernel, Fraction(0)) + count

    def merge(self, other: "FlopLedger") -> None:
        self.multiplications += other.multiplications
        for k, v in other.by_kernel.items():
            self.by_kernel[k] = self.by_kernel.get(k, Fraction(0)) + v

    def __add__(self, other: "FlopLedger") -> "FlopLedger":
        out = FlopLedger(self.multiplications, dict(self.by_kernel))
        out.merge(other)
        return out

    def as_float(self) -> float:
        return float(self.multiplications)


_F = Fraction
# (c3, c21, c12) for s^3, s^2 b, s b^2  (kernels.py:89-99)
MODELS_SB = {
    "naive_dense": (_F(1, 3), 1, 1),
    "sigma_naive": (0, 1, 3),
    "cholesky": (_F(1, 6), _F(1, 2), _F(1, 2)),
    "cholesky_with_factor": (_F(1, 6), 1, _F(1, 2)),
    "ldlt": (_F(1, 6), _F(1, 2), _F(1, 2)),
    "ldlt_with_factor": (_F(1, 6), 1, _F(1, 2)),
    "sigma_sparse": (0, _F(1, 2), 2),
    "sigma_sparse_alt": (0, 1, _F(3, 2)),
    "sigma_symmetric": (_F(1, 6), 1, _F(3, 2)),
}
# (c3, c21, c12) for m^3, m^2 n, m n^2 with m = s/2, n = b/2 (kernels.py:100-111)
MODELS_MN = {
    "parallel_inverse": (_F(8, 3), 4, 4),
    "sequential_inverse": (_F(4, 3), 5, 4),
    "block_lu": (_F(4, 3), 4, 5),
    "naive_lu": (_F(8, 3), _F(13, 2), 4),
    "parallel_inverse_with_factor": (_F(8, 3), 6, 4),
    "sequential_inverse_with_factor": (_F(4, 3), 5, 4),
    "block_lu_with_factor": (_F(4, 3), 5, 4),
    "naive_lu_with_factor": (_F(8, 3), _F(15, 2), 4),
    "symmetric_sparse": (_F(2, 3), 2, _F(5, 2)),
    "symmetric_sparse_with_factor": (_F(2, 3), 6, _F(5, 2)),
}
BLOCK_KERNELS = ("parallel_inverse", "sequential_inverse", "block_lu", "naive_lu")
HERMITIAN_KERNELS = ("cholesky", "symmetric_sparse")
KERNEL_NAMES = ("naive",) + BLOCK_KERNELS + ("cholesky", "ldlt", "symmetric_sparse")


def flop_model(kernel: str, m=None, n=None, s=None, b=None, c=None, t=None) -> Fraction:
    """Closed-form multiplication count of one kernel invocation (kernels.py:116-146)."""
    if kernel in MODELS_SB:
        if s is None or b is None:
            raise ValueError(f"kernel {kernel!r} needs sizes s and b")
        c3, c21, c12 = MODELS_SB[kernel]
        s, b = Fraction(s), Fraction(b)
        return Fraction(c3 * s**3 + c21 * s**2 * b + c12 * s * b**2)
    if kernel in MODELS_MN:
        if m is None or n is None:
            if s is None or b is None:
                raise ValueError(f"kernel {kernel!r} needs sizes (m, n) or (s, b)")
            m, n = Fraction(s, 2), Fraction(b, 2)
        c3, c21, c12 = MODELS_MN[kernel]
        m, n = Fraction(m), Fraction(n)
        return Fraction(c3 * m**3 + c21 * m**2 * n + c12 * m * n**2)
    if kernel == "dense_inverse":
        if c is None:
            raise ValueError("dense_inverse needs size c")
        return Fraction(c) ** 3
    if kernel == "gless_sandwich":
        if c is None:
            raise ValueError("gless_sandwich needs size c")
        return 2 * Fraction(c) ** 3
    if kernel == "offdiag_backsub":
        if t is None or c is None:
            raise ValueError("offdiag_backsub needs sizes t and c")
        t, c = Fraction(t), Fraction(c)
        return 2 * (t**2 * c + t * c**2)
    raise ValueError(f"unknown kernel {kernel!r}")


def _poly_sum(model, s, b, mn: bool) -> Fraction:
    """Exact sum of one polynomial model over arrays s, b (int64, exact via Python ints)."""
    if s.size == 0:
        return Fraction(0)
    s3 = int(np.sum(s.astype(object) ** 3))
    s2b = int(np.sum(s.astype(object) ** 2 * b.astype(object)))
    sb2 = int(np.sum(s.astype(object) * b.astype(object) ** 2))
    c3, c21, c12 = (Fraction(x) for x in model)
    if mn:
        c3, c21, c12 = c3 / 8, c21 / 8, c12 / 8
    return c3 * s3 + c21 * s2b + c12 * sb2


def plan_ledger(kind: np.ndarray, s: np.ndarray, b: np.ndarray, kernel: str = "naive", compute_gless: bool = True,
                sigma_hermitian: bool = False, sigma_mode: str = "auto") -> FlopLedger:
    """Ledger of one energy point, following solver.py:135-172 dispatch and the
    final-step charges (solver.py:388, 404, 410, 664).  kind: 0 leaf seed,
    1 upward merge, 2 downward merge, 3 final leaf step."""
    led = FlopLedger()
    kind = np.asarray(kind)
    s = np.asarray(s, dtype=np.int64)
    b = np.asarray(b, dtype=np.int64)
    fin = kind == 3
    elim = ~fin & (s > 0)
    split = elim & ((kind == 1) | (kind == 2))
    seed = elim & (kind == 0)
    wf = compute_gless

    def add(key, model, mask, mn=False):
        v = _poly_sum(model, s[mask], b[mask], mn)
        if mask.any():
            led.add(key, v)

    # A-kernel (solver.py:135-154)
    if kernel == "naive":
        add("naive_dense", MODELS_SB["naive_dense"], elim)
    elif kernel in BLOCK_KERNELS:
        add("naive_dense", MODELS_SB["naive_dense"], seed)
        key = kernel + ("_with_factor" if wf else "")
        add(key, MODELS_MN[key], split, mn=True)
    elif kernel == "ldlt":
        add("ldlt", MODELS_SB["ldlt_with_factor" if wf else "ldlt"], elim)
    elif kernel == "cholesky":
        add("cholesky", MODELS_SB["cholesky_with_factor" if wf else "cholesky"], elim)
    elif kernel == "symmetric_sparse":
        add("cholesky", MODELS_SB["cholesky_with_factor" if wf else "cholesky"], seed)
        add("symmetric_sparse", MODELS_MN["symmetric_sparse_with_factor" if wf else "symmetric_sparse"], split, mn=True)
    else:
        raise ValueError(f"unknown kernel {kernel!r}")
    # Sigma update (solver.py:157-172)
    if compute_gless:
        if sigma_mode != "general" and kernel in HERMITIAN_KERNELS and sigma_hermitian:
            add("sigma_symmetric", MODELS_SB["sigma_symmetric"], elim)
        elif sigma_mode != "general" and kernel in BLOCK_KERNELS:
            add("sigma_naive", MODELS_SB["sigma_naive"], seed)
            add("sigma_sparse", MODELS_SB["sigma_sparse"], split)
        else:
            add("sigma_naive", MODELS_SB["sigma_naive"], elim)
    # final leaf step: naive schur + sigma, inverse, sandwich (always naive)
    ffin = fin & (s > 0)
    add("naive_dense", MODELS_SB["naive_dense"], ffin)
    if compute_gless:
        add("sigma_naive", MODELS_SB["sigma_naive"], ffin)
    c = b[fin].astype(object)
    if fin.any():
        led.add("dense_inverse", Fraction(int(np.sum(c**3))))
        if compute_gless:
            led.add("gless_sandwich", Fraction(2 * int(np.sum(c**3))))
    return led
