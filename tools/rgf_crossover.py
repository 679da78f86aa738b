"""FIND vs RGF on the B200 (the paper's crossover question): energy
points/s of the GPU RGF path (paper_1104_0623_b200.rgf, find_dense_inverse / find_zgemm_batched) next
to the FIND path (solve_values), per BASELINE config.  One JSON line per config.

    python tools/rgf_crossover.py [--configs 0,1,2,3] [--chunk 8]
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1104_0623_b200 import Mesh, SparseOperator  # noqa: E402
from paper_1104_0623_b200.configs import config_problem  # noqa: E402
from paper_1104_0623_b200.plan import plan_for, release_workspaces  # noqa: E402
from paper_1104_0623_b200.rgf import rgf_batch  # noqa: E402
from paper_1104_0623_b200.solver import sigma_symmetry, solve_values  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="0,1,2,3")
ap.add_argument("--chunk", type=int, default=8, help="energy points per RGF batch")
a = ap.parse_args()
for c in [int(x) for x in a.configs.split(",")]:
    p = config_problem(c)
    mesh = Mesh(p.nx, p.ny)
    ne = p.energies.size
    sig = SparseOperator(p.sigma_csr())
    ops = [SparseOperator(p.a_csr(k)) for k in range(ne)]
    release_workspaces()
    rgf_batch(mesh, ops[:1], sig)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    gr_r, gl_r = [], []
    for k0 in range(0, ne, a.chunk):
        g1, g2, led = rgf_batch(mesh, ops[k0:k0 + a.chunk], sig)
        gr_r.append(g1)
        gl_r.append(g2)
    torch.cuda.synchronize()
    t_rgf = time.perf_counter() - t0
    torch.cuda.empty_cache()
    plan, _ = plan_for(p.nx, p.ny, p.indptr, p.indices)
    ssym = sigma_symmetry(p.sigma_csr())
    solve_values(plan, p.a_vals_all()[:1], p.s_vals, sigma_sym=ssym)
    t0 = time.perf_counter()
    gr_f, gl_f, tu, td = solve_values(plan, p.a_vals_all(), p.s_vals, sigma_sym=ssym)
    t_find = time.perf_counter() - t0
    gr_r, gl_r = np.concatenate(gr_r), np.concatenate(gl_r)
    rel = lambda x, y: float(np.max(np.abs(x - y)) / np.max(np.abs(y)))
    print(json.dumps({"config": c, "mesh": [p.nx, p.ny], "energies": ne,
                      "rgf_s": round(t_rgf, 4), "rgf_points_per_s": round(ne / t_rgf, 3),
                      "find_s": round(t_find, 4), "find_points_per_s": round(ne / t_find, 3),
                      "find_device_s": round(tu + td, 4), "rgf_W_per_energy": float(led["gr"].multiplications +
                                                                                     led["gless"].multiplications),
                      "find_W_per_energy": float(plan.native_work(0)),
                      "agree_gr": rel(gr_r, gr_f), "agree_gl": rel(gl_r, gl_f)}), flush=True)
    release_workspaces()
    torch.cuda.empty_cache()
