"""One warm-up + one timed FIND solve of a BASELINE config (for ncu launch lists / captures).

    python tools/profile_step.py [--config 1] [--energies 16]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1104_0623_b200.configs import config_problem  # noqa: E402
from paper_1104_0623_b200.plan import plan_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--energies", type=int, default=None)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
p = config_problem(a.config, a.energies)
plan, _ = plan_for(p.nx, p.ny, p.indptr, p.indices)
dev = torch.device("cuda", 0)
ad = torch.from_numpy(p.a_vals_all()).to(dev)
sd = torch.from_numpy(p.s_vals).to(dev)
gr = torch.empty((p.energies.size, p.n), dtype=torch.complex128, device=dev)
gl = torch.empty_like(gr)
ws = plan.workspace(p.energies.size, True, dev)
for _ in range(a.reps):
    plan.run(ad, sd, gr, gl, ws=ws, sigma_sym=-1)
plan.check_status(ws, p.energies.size)
torch.cuda.synchronize()
print("launches per solve", plan.launch_count(p.energies.size))
