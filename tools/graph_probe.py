"""Device time of one solve issued directly vs replayed from a captured CUDA graph.

    python tools/graph_probe.py [--config 1] [--reps 10]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1104_0623_b200.configs import config_problem  # noqa: E402
from paper_1104_0623_b200.plan import plan_for  # noqa: E402
from paper_1104_0623_b200.solver import sigma_symmetry  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--reps", type=int, default=10)
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
ssym = sigma_symmetry(p.sigma_csr())
stream = torch.cuda.Stream(dev)
with torch.cuda.stream(stream):
    for _ in range(3):
        plan.run(ad, sd, gr, gl, ws=ws, stream=stream, sigma_sym=ssym)
    torch.cuda.synchronize()
    ref = gr.clone()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(a.reps):
        plan.run(ad, sd, gr, gl, ws=ws, stream=stream, sigma_sym=ssym)
    e1.record(stream)
    torch.cuda.synchronize()
    direct = e0.elapsed_time(e1) / a.reps
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=stream):
    plan.run(ad, sd, gr, gl, ws=ws, stream=stream, sigma_sym=ssym)
torch.cuda.synchronize()
with torch.cuda.stream(stream):
    g.replay()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(a.reps):
        g.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    graph = e0.elapsed_time(e1) / a.reps
plan.check_status(ws, ne, stream)
print(f"config {a.config}: direct {direct:.3f} ms/solve, graph replay {graph:.3f} ms/solve, "
      f"identical {bool(torch.equal(gr, ref))}")
