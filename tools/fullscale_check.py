"""Full-scale run of a BASELINE config with independent sparse-LU spot checks.

    python tools/fullscale_check.py --config 2 [--energies 4] [--nodes 8]
Checks diag(G^r), diag(G^<) at sampled nodes against x = A^{-H} e_i from SuperLU
(G^r_ii = conj(x_i), G^<_ii = x^H Sigma^< x) and the sign structure of G^r / G^<.
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import scipy.sparse.linalg as spla  # noqa: E402

from paper_1104_0623_b200.configs import config_problem  # noqa: E402
from paper_1104_0623_b200.plan import plan_for  # noqa: E402
from paper_1104_0623_b200.solver import sigma_symmetry, solve_values  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--energies", type=int, default=None)
    ap.add_argument("--nodes", type=int, default=8)
    ap.add_argument("--check-energies", type=int, default=2)
    a = ap.parse_args()
    t0 = time.time()
    p = config_problem(a.config, a.energies)
    plan, tplan = plan_for(p.nx, p.ny, p.indptr, p.indices)
    t1 = time.time()
    gr, gl, tu, td = solve_values(plan, p.a_vals_all(), p.s_vals, sigma_sym=sigma_symmetry(p.sigma_csr()))
    t2 = time.time()
    res = {"config": a.config, "n": p.n, "energies": int(p.energies.size), "plan_s": tplan, "solve_wall_s": t2 - t1,
           "device_s": tu + td, "im_gr_negative": bool(np.all(gr.imag < 0)),
           "gl_real_rel": float(np.max(np.abs(gl.real)) / np.max(np.abs(gl))),
           "gl_imag_min_rel": float(np.min(gl.imag) / np.max(np.abs(gl)))}
    rng = np.random.default_rng(0)
    sig = p.sigma_csr()
    worst_gr = worst_gl = 0.0
    ks = np.unique(np.linspace(0, p.energies.size - 1, a.check_energies).round().astype(int))
    for k in ks:
        lu = spla.splu(p.a_csr(int(k)).conj().T.tocsc())
        nodes = rng.choice(p.n, a.nodes, replace=False)
        nodes[:2] = [0, p.n - 1]
        for i in nodes:
            e = np.zeros(p.n, complex)
            e[i] = 1.0
            x = lu.solve(e)
            worst_gr = max(worst_gr, abs(gr[k, i] - np.conj(x[i])) / np.max(np.abs(gr[k])))
            worst_gl = max(worst_gl, abs(gl[k, i] - np.vdot(x, sig @ x)) / np.max(np.abs(gl[k])))
    res.update({"spot_rel_gr": worst_gr, "spot_rel_gl": worst_gl, "checked_energies": ks.tolist(),
                "total_s": time.time() - t0})
    print("RESULT", json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
