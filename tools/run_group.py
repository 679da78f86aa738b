"""One full cfg solve (inputs, arenas), then the launch groups given by --groups run alone:
the target of a focused ncu capture (`-k regex:<kernel> -s <launches of that kernel per solve>`);
without --groups, one solve (the launch list of `ncu --metrics ...`).

    python tools/run_group.py --config 1 --groups 104 108
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
ap.add_argument("--groups", type=int, nargs="*", default=[])
ap.add_argument("--no-full", action="store_true", help="skip the full solve (inputs of the groups then stale)")
ap.add_argument("--energies", type=int, default=0, help="first N energy points of the config (0: all)")
ap.add_argument("--profile-groups", action="store_true",
                help="cudaProfilerStart/Stop around the group runs (ncu --profile-from-start off)")
a = ap.parse_args()
p = config_problem(a.config, a.energies or None)
plan, _ = plan_for(p.nx, p.ny, p.indptr, p.indices)
dev = torch.device("cuda", 0)
ne = p.energies.size
ad = torch.from_numpy(p.a_vals_all()).to(dev)
sd = torch.from_numpy(p.s_vals).to(dev)
gr = torch.empty((ne, p.n), dtype=torch.complex128, device=dev)
gl = torch.empty_like(gr)
ws = plan.workspace(ne, True, dev)
if not a.no_full:
    plan.run(ad, sd, gr, gl, ws=ws, sigma_sym=-1)
torch.cuda.synchronize()
if a.profile_groups:
    torch.cuda.profiler.start()
for gi in a.groups:
    plan.run(ad, sd, gr, gl, ws=ws, sigma_sym=-1, groups=(gi, gi + 1))
    torch.cuda.synchronize()
if a.profile_groups:
    torch.cuda.profiler.stop()
print("ok")
