"""Error level of the GPU path against the full-size reference fixtures (tests/golden/full_cfg*.npz)
under the current FIND_B200_* environment; one JSON line per config.

    FIND_B200_NB=16 python tools/err_probe.py 1 2 [--sym 0]
"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402

from paper_1104_0623_b200.configs import config_problem  # noqa: E402
from paper_1104_0623_b200.plan import Plan  # noqa: E402
from paper_1104_0623_b200.solver import sigma_symmetry, solve_values  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
sym_override = None
if "--sym" in sys.argv:
    sym_override = int(sys.argv[sys.argv.index("--sym") + 1])
    args = [a for a in args if a != str(sym_override)]
env = {k: v for k, v in os.environ.items() if k.startswith("FIND_B200")}
for c in map(int, args):
    f = np.load(Path(__file__).resolve().parent.parent / "tests" / "golden" / f"full_cfg{c}.npz")
    p = config_problem(c)
    ks = [int(k) for k in f["energy_idx"]]
    plan = Plan(p.nx, p.ny, p.indptr, p.indices)
    a = p.a_vals_all()[ks]
    sym = sigma_symmetry(p.sigma_csr()) if sym_override is None else sym_override
    gr, gl, _, _ = solve_values(plan, a, p.s_vals, sigma_sym=sym)
    eg = [float(np.abs(gr[i] - f["gr"][i]).max() / np.abs(f["gr"][i]).max()) for i in range(len(ks))]
    el = [float(np.abs(gl[i] - f["gl"][i]).max() / np.abs(f["gl"][i]).max()) for i in range(len(ks))]
    i = int(np.argmax(el))
    d = np.abs(gl[i] - f["gl"][i])
    worst = int(np.argmax(d))
    rows = np.bincount(np.arange(p.n) // p.nx, weights=d, minlength=p.ny)
    print(json.dumps({"config": c, "env": env, "sym": sym, "gr": max(eg), "gl": max(el), "gr_each": eg, "gl_each": el,
                      "worst_node_xy": [worst % p.nx, worst // p.nx],
                      "max_abs_gl": float(np.abs(f["gl"][i]).max()), "max_abs_gr": float(np.abs(f["gr"]).max()),
                      "err_by_row_top": np.argsort(-rows)[:5].tolist()}), flush=True)
