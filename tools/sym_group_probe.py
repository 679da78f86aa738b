"""Which output entries of one downward launch group change when the symmetric (mirrored) R
mode is switched on for that group alone?  Runs groups [0, g] twice on the same inputs
(general mode; general up to g-1 then symmetric for g), diffs the block arenas, maps every
differing entry to its elimination's U / R block and prints the pattern, plus the skewness
of the general-mode R blocks.  Needs FIND_B200_RSYM_DOWN=1 (downward symmetric mode).

    FIND_B200_RSYM_DOWN=1 python tools/sym_group_probe.py 32 128 27
"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1104_0623_b200 import _native  # noqa: E402
from paper_1104_0623_b200.configs import build_problem  # noqa: E402
from paper_1104_0623_b200.plan import Plan  # noqa: E402

nx, ny, gsel = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
p = build_problem(nx, ny, [1.7], seed=3, stencil=5, vamp=1.0)
plan = Plan(p.nx, p.ny, p.indptr, p.indices)
L = _native.lib()
ne = plan.info["n_elims"]
oa = np.zeros(ne, np.int32)
oo = np.zeros(ne, np.int64)
L.find_plan_elim_out(plan.handle, oa.ctypes.data_as(C.POINTER(C.c_int32)), oo.ctypes.data_as(C.POINTER(C.c_int64)))
ae = np.zeros(4, np.int64)
L.find_plan_arena_elems(plan.handle, ae.ctypes.data_as(C.POINTER(C.c_int64)))
dev = torch.device("cuda", 0)
a = torch.from_numpy(p.a_vals_all()).to(dev)
s = torch.from_numpy(p.s_vals).to(dev)
g = plan.groups
start = np.concatenate([[0], np.cumsum(g["count"])])
print("group", gsel, "pass", g["pass"][gsel], "level", g["level"][gsel], "path", g["path"][gsel], "count",
      g["count"][gsel], "max_s", g["max_s"][gsel], "max_b", g["max_b"][gsel])


def run(sym_last):
    gr = torch.empty((1, p.n), dtype=torch.complex128, device=dev)
    gl = torch.empty_like(gr)
    ws = plan.workspace(1, True, dev)
    ws.zero_()
    plan.run(a, s, gr, gl, ws=ws, groups=(0, gsel), sigma_sym=0)
    plan.run(a, s, gr, gl, ws=ws, groups=(gsel, gsel + 1), sigma_sym=sym_last)
    torch.cuda.synchronize()
    plan.check_status(ws, 1)
    base = 256
    arenas = []
    for k in range(4):
        nb = int(ae[k]) * 16
        arenas.append(ws[base:base + nb].view(torch.complex128).cpu().numpy().copy())
        base += nb
    return arenas


A = run(0)
B = run(-1)
for k in range(4):
    d = np.abs(A[k] - B[k])
    if d.size and d.max() > 0:
        print("arena", k, "entries differing", int((d > 0).sum()), "max", d.max())
for e in range(start[gsel], start[gsel + 1]):
    k = int(oa[e])
    if k < 0:
        continue
    b = int(plan.b[e])
    off = int(oo[e])
    U0 = A[k][off:off + b * b].reshape(b, b)
    R0 = A[k][off + b * b:off + 2 * b * b].reshape(b, b)
    R1 = B[k][off + b * b:off + 2 * b * b].reshape(b, b)
    U1 = B[k][off:off + b * b].reshape(b, b)
    sk = np.abs(R0 + R0.conj().T).max() / max(np.abs(R0).max(), 1e-300)
    dr = np.abs(R0 - R1)
    print(f"elim {e} label {plan.label[e]} kind {plan.kind[e]} s {plan.s[e]} b {b} arena {k} off {off}: "
          f"skew(R_general) {sk:.2e} max|R| {np.abs(R0).max():.2e} max|dR| {dr.max():.2e} max|dU| "
          f"{np.abs(U0 - U1).max():.2e}")
    if dr.max() > 1e-12 * np.abs(R0).max():
        rows, cols = np.nonzero(dr > 1e-12 * np.abs(R0).max())
        print("   differing R entries (sorted-B positions):", list(zip(rows.tolist(), cols.tolist()))[:40])
        asym = np.abs(R0 + R0.conj().T)
        rr, cc = np.nonzero(asym > 1e-10 * np.abs(R0).max())
        print("   general R non-skew entries:", list(zip(rr.tolist(), cc.tolist()))[:40])
