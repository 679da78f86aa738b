"""Device time of whole FIND solves (all launch groups, concurrent lanes as in production), CUDA events:
the quick A/B for scheduling switches.

    python tools/step_time.py --config 4 --energies 4 [--reps 3] [--graph]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1104_0623_b200.configs import config_problem  # noqa: E402
from paper_1104_0623_b200.plan import plan_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--energies", type=int, default=4)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
p = config_problem(a.config, a.energies)
plan, _ = plan_for(p.nx, p.ny, p.indptr, p.indices)
dev = torch.device("cuda", 0)
ne = p.energies.size
ad = torch.from_numpy(p.a_vals_all()).to(dev)
sd = torch.from_numpy(p.s_vals).to(dev)
gr = torch.empty((ne, p.n), dtype=torch.complex128, device=dev)
gl = torch.empty_like(gr)
ws = plan.workspace(ne, True, dev)
plan.run(ad, sd, gr, gl, ws=ws, sigma_sym=-1)
torch.cuda.synchronize()
ms = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    plan.run(ad, sd, gr, gl, ws=ws, sigma_sym=-1)
    e1.record()
    torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
plan.check_status(ws, ne)
print(f"cfg{a.config} x{ne}: solve ms {[round(x, 1) for x in ms]}  best {min(ms):.1f}  -> {ne / min(ms) * 1e3:.3f} energy points/s")
