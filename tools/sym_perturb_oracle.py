"""Sensitivity of diag(G^<) to roundoff-sized perturbations of the downward R blocks, in the CPU
oracle (reference algorithm, LAPACK): each downward sigma_update output R is replaced by
  lower-mirror : tril(R) - tril(R,-1)^H               (the symmetric mode)
  rand-skew    : R + eps * |R| .* (skew-Hermitian noise)    (eps = 2^-52, elementwise relative)
  rand-herm    : R + eps * |R| .* (Hermitian noise)
  rand-any     : R + eps * |R| .* (complex noise, no symmetry)
and diag(G^<) is compared with the unmodified oracle.  If elementwise roundoff-sized noise moves
the result as much as the mirror does, the mirror is within the recurrence's own conditioning.

    python tools/sym_perturb_oracle.py [nx ny]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import find_oracle as fo  # noqa: E402
from paper_1104_0623_b200.configs import build_problem  # noqa: E402

cases = [(int(sys.argv[1]), int(sys.argv[2]))] if len(sys.argv) > 2 else [(32, 128), (64, 256)]
eps = 2.0 ** -52
for nx, ny in cases:
    p = build_problem(nx, ny, [1.7], seed=3, stencil=5, vamp=1.0)
    a = p.a_csr(0)
    sg = p.sigma_csr()
    o = fo.FindOracle(p.nx, p.ny, a)
    base = o.solve(a, sg)
    for mode in ("lower-mirror", "rand-skew", "rand-herm", "rand-any"):
        rng = np.random.default_rng(11)
        orig = fo.sigma_update

        def su(sss, ssb, sbs, sbb, l_fac, ledger, orig=orig, mode=mode, rng=rng):
            r = orig(sss, ssb, sbs, sbb, l_fac, ledger)
            if mode == "lower-mirror":
                return np.tril(r) - np.tril(r, -1).conj().T
            z = rng.uniform(-1, 1, r.shape) + 1j * rng.uniform(-1, 1, r.shape)
            if mode == "rand-skew":
                z = 0.5 * (z - z.conj().T)
            elif mode == "rand-herm":
                z = 0.5 * (z + z.conj().T)
            return r + eps * np.abs(r) * z

        oe = o._eliminate

        def elim(a_, sg_, left, right, ul, ur, rl, rr, s_set, label, want, led, rtol, oe=oe, su=su, orig=orig):
            if label < 0:
                fo.sigma_update = su
            try:
                return oe(a_, sg_, left, right, ul, ur, rl, rr, s_set, label, want, led, rtol)
            finally:
                fo.sigma_update = orig

        o._eliminate = elim
        r = o.solve(a, sg)
        o._eliminate = oe
        d = r.gless_diag - base.gless_diag
        sc = np.abs(base.gless_diag).max()
        print(f"{nx}x{ny} {mode:12s} diag(G^<) change: max|d|/max|ref| {np.abs(d).max() / sc:.2e}"
              f"  (imag part {np.abs(d.imag).max() / sc:.2e}, real part {np.abs(d.real).max() / sc:.2e})", flush=True)
