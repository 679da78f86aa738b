"""Launch timeline of one solve (CUDA events around every launch, all side streams):
per phase its span, the busiest group chain, and the launches on that chain.

    python tools/timeline.py [--config 1] [--out timeline.json]
"""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1104_0623_b200 import _native  # noqa: E402
from paper_1104_0623_b200.configs import config_problem  # noqa: E402
from paper_1104_0623_b200.plan import Plan, plan_for  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--out", default="")
a = ap.parse_args()
p = config_problem(a.config)
plan, _ = plan_for(p.nx, p.ny, p.indptr, p.indices)
dev = torch.device("cuda", 0)
ne = p.energies.size
ad = torch.from_numpy(p.a_vals_all()).to(dev)
sd = torch.from_numpy(p.s_vals).to(dev)
gr = torch.empty((ne, p.n), dtype=torch.complex128, device=dev)
gl = torch.empty_like(gr)
ws = plan.workspace(ne, True, dev)
L = _native.lib()
for _ in range(2):
    plan.run(ad, sd, gr, gl, ws=ws, sigma_sym=-1)
torch.cuda.synchronize()
L.find_solve_timing_enable(1)
plan.run(ad, sd, gr, gl, ws=ws, sigma_sym=-1)
torch.cuda.synchronize()
L.find_solve_timing_enable(0)
n = int(L.find_solve_timing_read2(None, None, None, None, 0))
kk = (C.c_int32 * n)()
gg = (C.c_int32 * n)()
t0 = (C.c_float * n)()
t1 = (C.c_float * n)()
L.find_solve_timing_read2(kk, gg, t0, t1, n)
kk, gg, t0, t1 = np.array(kk), np.array(gg), np.array(t0), np.array(t1)
ph = plan.group_phases()
g = plan.groups
print(f"solve span {t1.max() - t0.min():.2f} ms, {n} launches, sum of durations {np.sum(t1 - t0):.2f} ms")
rows = []
for phase in np.unique(ph):
    sel = np.isin(gg, np.nonzero(ph == phase)[0])
    if not sel.any():
        continue
    span = t1[sel].max() - t0[sel].min()
    gspan = {}
    for gi in np.unique(gg[sel]):
        m = gg == gi
        gspan[int(gi)] = (float(t0[m].min()), float(t1[m].max()), float(np.sum(t1[m] - t0[m])), int(m.sum()))
    crit = max(gspan, key=lambda x: gspan[x][1] - gspan[x][0])
    c = gspan[crit]
    rows.append({"phase": int(phase), "span_ms": float(span), "groups": len(gspan), "crit_group": crit,
                 "crit_span": c[1] - c[0], "crit_busy": c[2], "crit_launches": c[3],
                 "crit_s": int(g["max_s"][crit]), "crit_b": int(g["max_b"][crit]), "crit_n_elims": int(g["count"][crit])})
    print(f"phase {phase:2d} span {span:6.2f} ms  groups {len(gspan):2d}  critical g{crit} "
          f"(s<={g['max_s'][crit]}, b<={g['max_b'][crit]}, {g['count'][crit]} elims): span {c[1] - c[0]:.2f} ms, "
          f"busy {c[2]:.2f} ms over {c[3]} launches")
if a.out:
    Path(a.out).write_text(json.dumps({"phases": rows, "launches": [
        {"kind": Plan.KIND_NAMES[int(k)], "group": int(x), "t0": float(b), "t1": float(e)} for k, x, b, e in zip(kk, gg, t0, t1)]}))
