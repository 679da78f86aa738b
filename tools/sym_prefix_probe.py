"""Where does the downward symmetric-R mode first diverge from the general mode?  For every
downward launch group g, groups [0, g] are run in ONE call twice (general; symmetric with
FIND_B200_RSYM_DOWN=1 in the environment), and the R blocks that group g wrote are compared;
the first groups with a relative difference above 1e-10 are printed with their shapes, plus the
skewness of the general-mode blocks.

    FIND_B200_RSYM_DOWN=1 python tools/sym_prefix_probe.py 64 256
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

nx, ny = int(sys.argv[1]), int(sys.argv[2])
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
fd = plan.first_down_group


def run(g_end, sym):
    gr = torch.empty((1, p.n), dtype=torch.complex128, device=dev)
    gl = torch.empty_like(gr)
    ws = plan.workspace(1, True, dev)
    ws.zero_()
    plan.run(a, s, gr, gl, ws=ws, groups=(0, g_end), sigma_sym=sym)
    torch.cuda.synchronize()
    plan.check_status(ws, 1)
    base, arenas = 256, []
    for k in range(4):
        nb = int(ae[k]) * 16
        arenas.append(ws[base:base + nb].view(torch.complex128).cpu().numpy().copy())
        base += nb
    return arenas, gl.cpu().numpy()[0]


shown = 0
for gi in range(fd, len(g["count"])):
    if g["pass"][gi] != 1:
        continue
    A, _ = run(gi + 1, 0)
    B, _ = run(gi + 1, -1)
    worst = (0.0, None)
    for e in range(start[gi], start[gi + 1]):
        k = int(oa[e])
        if k < 0:
            continue
        b = int(plan.b[e])
        off = int(oo[e])
        R0 = A[k][off + b * b:off + 2 * b * b].reshape(b, b)
        R1 = B[k][off + b * b:off + 2 * b * b].reshape(b, b)
        rel = np.abs(R0 - R1).max() / max(np.abs(R0).max(), 1e-300)
        sk = np.abs(R0 + R0.conj().T).max() / max(np.abs(R0).max(), 1e-300)
        if rel > worst[0]:
            worst = (rel, (e, int(plan.s[e]), b, sk, int(plan.label[e])))
    print(f"g{gi} L{g['level'][gi]} path{g['path'][gi]} n={g['count'][gi]} s<={g['max_s'][gi]} b<={g['max_b'][gi]}: "
          f"max rel dR {worst[0]:.2e} {worst[1]}", flush=True)
    if worst[0] > 1e-10:
        shown += 1
        if shown >= 4:
            break
