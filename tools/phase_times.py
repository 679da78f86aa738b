"""Device time of every phase of one solve (groups of a phase run together), for
comparing schedules: python tools/phase_times.py [--config 1] [--per-group]."""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1104_0623_b200.configs import config_problem  # noqa: E402
from paper_1104_0623_b200.plan import plan_for  # noqa: E402
from paper_1104_0623_b200.workmodel import executed_cmacs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--energies", type=int, default=None)
ap.add_argument("--out", default="")
ap.add_argument("--per-group", action="store_true", help="time every group alone (serialised)")
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
ph = plan.group_phases()
bounds = [0] + [i for i in range(1, len(ph)) if ph[i] != ph[i - 1]] + [len(ph)]
if a.per_group:
    bounds = list(range(len(ph) + 1))
work = executed_cmacs(plan, -1)
for rep in range(3):
    evs = []
    for k in range(len(bounds) - 1):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.run(ad, sd, gr, gl, ws=ws, sigma_sym=-1, groups=(bounds[k], bounds[k + 1]))
        e1.record()
        evs.append((e0, e1))
    torch.cuda.synchronize()
if not os.environ.get("FIND_B200_SKIP"):
    plan.check_status(ws, ne)
rows = []
g = plan.groups
for k in range(len(bounds) - 1):
    gs = range(bounds[k], bounds[k + 1])
    ms = evs[k][0].elapsed_time(evs[k][1])
    cm = sum(v for (gi, kk), v in work.items() if gi in gs) * ne
    rows.append({"phase": int(ph[bounds[k]]), "pass": int(g["pass"][bounds[k]]), "level": int(g["level"][bounds[k]]),
                 "groups": len(gs), "paths": [int(g["path"][i]) for i in gs],
                 "mean_s": int(np.mean(plan.s[int(np.sum(g["count"][:gs[0]])):int(np.sum(g["count"][:gs[-1] + 1]))])),
                 "max_s": int(max(g["max_s"][i] for i in gs)), "max_b": int(max(g["max_b"][i] for i in gs)),
                 "elims": int(sum(g["count"][i] for i in gs)), "ms": round(ms, 3),
                 "tflops": round(8 * cm / (ms * 1e-3) / 1e12, 2)})
tot = sum(r["ms"] for r in rows)
print("total ms", round(tot, 2))
for r in rows:
    print(json.dumps(r))
if a.out:
    Path(a.out).write_text(json.dumps({"total_ms": tot, "phases": rows}, indent=1))
