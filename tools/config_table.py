"""Throughput on every BASELINE config (energy points/s, FP64 TFLOP/s on the reference ledger W),
through solve_values (energy chunks sized to free HBM; device time = CUDA events around the
level launches, wall = the whole call incl. H2D / D2H).  One JSON line per config.

    python tools/config_table.py [--configs 0,1,2,3,4] [--offdiag3] [--energies N]
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402

from paper_1104_0623_b200.configs import CONFIGS, config_problem  # noqa: E402
from paper_1104_0623_b200.plan import plan_for  # noqa: E402
from paper_1104_0623_b200.solver import sigma_symmetry, solve_values  # noqa: E402

FP64_PEAK = 37.19
ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="0,1,2,3,4")
ap.add_argument("--offdiag3", action="store_true", help="config 3 also with compute_offdiag (its BASELINE outputs)")
ap.add_argument("--energies", type=int, default=None, help="cap the energy points per config")
a = ap.parse_args()
for c in [int(x) for x in a.configs.split(",")]:
    t0 = time.perf_counter()
    p = config_problem(c, a.energies)
    plan, tb = plan_for(p.nx, p.ny, p.indptr, p.indices)
    ne = p.energies.size
    vals = p.a_vals_all()
    ssym = sigma_symmetry(p.sigma_csr())
    for _ in range(2):  # warm-up: eager, then the CUDA-graph capture (timed calls replay)
        solve_values(plan, vals, p.s_vals, sigma_sym=ssym)
    runs = [False, True] if (c == 3 and a.offdiag3) else [False]
    for off in runs:
        out = {}
        w0 = time.perf_counter()
        gr, gl, tu, td = solve_values(plan, vals, p.s_vals, sigma_sym=ssym, compute_offdiag=off, offdiag_out=out)
        wall = time.perf_counter() - w0
        dev = tu + td
        W = float(plan.native_work(0))
        line = {"config": c, "mesh": [p.nx, p.ny], "stencil": CONFIGS[c].stencil, "energies": ne,
                "compute_offdiag": off, "n_pairs": int(out["gr"].shape[1]) if off else 0,
                "device_s": round(dev, 4), "wall_s": round(wall, 4),
                "energy_points_per_s_device": round(ne / dev, 3), "energy_points_per_s_wall": round(ne / wall, 3),
                "W_per_energy": W, "fp64_tflops": round(8 * W * ne / dev / 1e12, 3),
                "fp64_frac_of_peak": round(8 * W * ne / dev / 1e12 / FP64_PEAK, 4),
                "plan_build_s": round(tb, 2), "gr_imag_negative": bool(np.all(gr.imag < 0))}
        print(json.dumps(line), flush=True)
