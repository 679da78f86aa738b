"""Find the smallest mesh where diag(G^<) disagrees with sparse-LU spot checks."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import scipy.sparse.linalg as spla  # noqa: E402

from paper_1104_0623_b200.configs import build_problem  # noqa: E402
from paper_1104_0623_b200.plan import Plan  # noqa: E402
from paper_1104_0623_b200.solver import solve_values  # noqa: E402


def check(nx, ny, vamp, sym, seed=3):
    p = build_problem(nx, ny, [1.7], seed=seed, stencil=5, vamp=vamp)
    plan = Plan(p.nx, p.ny, p.indptr, p.indices)
    gr, gl, _, _ = solve_values(plan, p.a_vals_all(), p.s_vals, sigma_sym=sym)
    lu = spla.splu(p.a_csr(0).conj().T.tocsc())
    sig = p.sigma_csr()
    worst = 0.0
    worst_gr = 0.0
    rng = np.random.default_rng(1)
    for i in list(rng.choice(p.n, 12, replace=False)) + [0, p.n - 1]:
        e = np.zeros(p.n, complex)
        e[i] = 1
        x = lu.solve(e)
        worst = max(worst, abs(gl[0, i] - np.vdot(x, sig @ x)) / np.max(np.abs(gl[0])))
        worst_gr = max(worst_gr, abs(gr[0, i] - np.conj(x[i])) / np.max(np.abs(gr[0])))
    return worst_gr, worst, float(np.max(np.abs(gl.real)) / np.max(np.abs(gl)))


for nx, ny in [(32, 128), (64, 256), (128, 512), (256, 256), (256, 512), (256, 1024)]:
    for vamp in (1.0,):
        for sym in (-1, 0):
            r = check(nx, ny, vamp, sym)
            print(nx, ny, vamp, sym, "gr %.1e gl %.1e realpart %.1e" % r, flush=True)
