"""Compare the arena contents (stored U/R blocks) of the general and the
skew-Hermitian-mirror R modes; report skewness of the general-mode R."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1104_0623_b200.configs import build_problem  # noqa: E402
from paper_1104_0623_b200.plan import Plan  # noqa: E402

nx, ny = int(sys.argv[1]), int(sys.argv[2])
p = build_problem(nx, ny, [1.7], seed=3, stencil=5, vamp=1.0)
plan = Plan(p.nx, p.ny, p.indptr, p.indices)
dev = torch.device("cuda", 0)
a = torch.from_numpy(p.a_vals_all()).to(dev)
s = torch.from_numpy(p.s_vals).to(dev)
out = {}
for sym in (0, -1):
    gr = torch.empty((1, p.n), dtype=torch.complex128, device=dev)
    gl = torch.empty_like(gr)
    ws = plan.workspace(1, True, dev)
    ws.zero_()
    plan.run(a, s, gr, gl, ws=ws, groups=(0, plan.first_down_group), sigma_sym=sym)
    plan.check_status(ws, 1)
    up = plan.info["up_arena_elems"]
    arena = ws[256:256 + up * 16].view(torch.complex128).cpu().numpy().copy()
    out[sym] = arena
d = np.abs(out[0] - out[-1])
print("up arena max |gen - sym|", d.max(), "max |arena|", np.abs(out[0]).max(), "argmax", int(d.argmax()), "of", d.size)
idx = np.argsort(-d)[:10]
print("top diffs", [(int(i), float(d[i]), complex(out[0][i]), complex(out[-1][i])) for i in idx[:5]])

# mixed modes: sym on up only / down only
res = {}
for up_sym, down_sym in ((0, 0), (-1, 0), (0, -1), (-1, -1)):
    gr = torch.empty((1, p.n), dtype=torch.complex128, device=dev)
    gl = torch.empty_like(gr)
    ws = plan.workspace(1, True, dev)
    plan.run(a, s, gr, gl, ws=ws, groups=(0, plan.first_down_group), sigma_sym=up_sym)
    plan.run(a, s, gr, gl, ws=ws, groups=(plan.first_down_group, -1), sigma_sym=down_sym)
    plan.check_status(ws, 1)
    res[(up_sym, down_sym)] = gl.cpu().numpy()[0]
ref = res[(0, 0)]
for k, v in res.items():
    err = np.abs(v - ref) / np.abs(ref).max()
    print(k, "max rel diff vs general", err.max(), "worst node", int(err.argmax()), "xy", int(err.argmax()) % nx, int(err.argmax()) // nx)
# per group: which groups in the down pass break it?  toggle sym per group
g = plan.groups
fd = plan.first_down_group
worst = []
for gi in range(fd, len(g["count"])):
    gr = torch.empty((1, p.n), dtype=torch.complex128, device=dev)
    gl = torch.empty_like(gr)
    ws = plan.workspace(1, True, dev)
    plan.run(a, s, gr, gl, ws=ws, groups=(0, gi), sigma_sym=0)
    plan.run(a, s, gr, gl, ws=ws, groups=(gi, gi + 1), sigma_sym=-1)
    plan.run(a, s, gr, gl, ws=ws, groups=(gi + 1, -1), sigma_sym=0)
    plan.check_status(ws, 1)
    e = float(np.abs(gl.cpu().numpy()[0] - ref).max() / np.abs(ref).max())
    worst.append((e, gi, int(g["pass"][gi]), int(g["level"][gi]), int(g["path"][gi]), int(g["count"][gi]), int(g["max_s"][gi]), int(g["max_b"][gi])))
for w in sorted(worst, reverse=True)[:8]:
    print("sym only in group: err %.2e g%d pass%d L%d path%d n=%d s<=%d b<=%d" % w)
