"""Root cause of the downward symmetric-R drift, in the CPU oracle (reference algorithm, LAPACK):
the downward Sigma updates (sigma_update, kernels.py:383-392) are replaced by
  lower-mirror: the lower triangle of R with its conjugate mirrored above (the GPU's symmetric mode)
  avg:          the skew-Hermitian projection (R - R^H) / 2
and diag(G^<) is compared with the unmodified oracle.  Writes nothing; prints one line per case.

    python tools/sym_mirror_oracle.py
"""
import numpy as np, sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from oracle import find_oracle as fo
from paper_1104_0623_b200.configs import build_problem
for nx, ny in [(32,128),(64,256)]:
    p = build_problem(nx, ny, [1.7], seed=3, stencil=5, vamp=1.0)
    a = p.a_csr(0); sg = p.sigma_csr()
    o = fo.FindOracle(p.nx, p.ny, a)
    base = o.solve(a, sg)
    for mode in ('lower-mirror', 'avg'):
        orig = fo.sigma_update
        def su(sss, ssb, sbs, sbb, l_fac, ledger, orig=orig, mode=mode):
            r = orig(sss, ssb, sbs, sbb, l_fac, ledger)
            if mode == 'avg':
                return 0.5 * (r - r.conj().T)
            lo = np.tril(r)
            return lo - np.tril(r, -1).conj().T
        # apply only to downward eliminations: label < 0 -> patch _eliminate
        oe = o._eliminate
        def elim(a_, sg_, left, right, ul, ur, rl, rr, s_set, label, want, led, rtol, oe=oe):
            if label < 0:
                fo.sigma_update = su
            try:
                return oe(a_, sg_, left, right, ul, ur, rl, rr, s_set, label, want, led, rtol)
            finally:
                fo.sigma_update = orig
        o._eliminate = elim
        r = o.solve(a, sg)
        o._eliminate = oe
        print(nx, ny, mode, 'gl diff vs plain oracle %.2e' % (np.abs(r.gless_diag - base.gless_diag).max() / np.abs(base.gless_diag).max()), flush=True)
