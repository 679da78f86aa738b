"""Serialized per-group profile of one solve: every launch group run alone (in plan
order, so data dependencies hold), each launch timed with CUDA events; prints per
group its shape, device ms, executed TFLOP/s and the per-kind split.

    python tools/group_kinds.py [--config 1] [--out groups.json] [--top 25]
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
from paper_1104_0623_b200.workmodel import executed_cmacs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--energies", type=int, default=None)
ap.add_argument("--out", default="")
ap.add_argument("--top", type=int, default=25)
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
L = _native.lib()
ng = len(plan.groups["count"])
for _ in range(2):
    plan.run(ad, sd, gr, gl, ws=ws, sigma_sym=-1)
torch.cuda.synchronize()
L.find_solve_timing_enable(1)
for gi in range(ng):
    plan.run(ad, sd, gr, gl, ws=ws, sigma_sym=-1, groups=(gi, gi + 1))
    torch.cuda.synchronize()
L.find_solve_timing_enable(0)
n = int(L.find_solve_timing_read(None, None, None, 0))
kk = (C.c_int32 * n)()
gg = (C.c_int32 * n)()
ms = (C.c_float * n)()
L.find_solve_timing_read(kk, gg, ms, n)
kk, gg, ms = np.array(kk), np.array(gg), np.array(ms)
work = executed_cmacs(plan, -1)
g = plan.groups
ph = plan.group_phases()
rows = []
for gi in range(ng):
    m = gg == gi
    kinds = {}
    for k, t in zip(kk[m], ms[m]):
        kinds[Plan.KIND_NAMES[int(k)]] = kinds.get(Plan.KIND_NAMES[int(k)], 0.0) + float(t)
    tot = float(ms[m].sum())
    cm = sum(v for (gj, _), v in work.items() if gj == gi) * ne
    rows.append({"group": gi, "phase": int(ph[gi]), "pass": int(g["pass"][gi]), "level": int(g["level"][gi]),
                 "path": int(g["path"][gi]), "elims": int(g["count"][gi]), "max_s": int(g["max_s"][gi]),
                 "max_b": int(g["max_b"][gi]), "launches": int(m.sum()), "ms": round(tot, 3),
                 "tflops": round(8 * cm / max(tot, 1e-9) / 1e9, 2),
                 "kinds": {k: round(v, 3) for k, v in sorted(kinds.items(), key=lambda x: -x[1])}})
total = sum(r["ms"] for r in rows)
print(f"serialized total {total:.2f} ms over {ng} groups, {n} launches")
by_kind = {}
for r in rows:
    for k, v in r["kinds"].items():
        by_kind[k] = by_kind.get(k, 0.0) + v
print("by kind:", json.dumps({k: round(v, 2) for k, v in sorted(by_kind.items(), key=lambda x: -x[1])}))
near = [r for r in rows if r["level"] <= 4 and r["pass"] in (0, 1)]
near_ms = sum(r["ms"] for r in near)
near_tf = sum(r["tflops"] * r["ms"] for r in near) / near_ms if near_ms else 0.0
near_root = {"config": a.config, "energies": ne, "levels": "upward 1-4 + downward 1-4", "groups": len(near),
             "ms_serialized": round(near_ms, 3), "tflops": round(near_tf, 3), "frac_fp64_peak": round(near_tf / 37.19, 4)}
print("near_root", json.dumps(near_root))
for r in sorted(rows, key=lambda r: -r["ms"])[: a.top]:
    print(json.dumps(r))
if a.out:
    Path(a.out).write_text(json.dumps({"total_ms": total, "by_kind": by_kind, "near_root": near_root, "groups": rows},
                                      indent=1))
