import os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_1104_0623_b200 import Mesh, SolverConfig, SparseOperator, solve_batch
from paper_1104_0623_b200 import solver as S
from paper_1104_0623_b200.configs import config_problem
p = config_problem(1)
mesh = Mesh(p.nx, p.ny)
ops = [SparseOperator(p.a_csr(k)) for k in range(16)]
sig = SparseOperator(p.sigma_csr())
conf = SolverConfig()
orig = S.solve_values
tm = {}
def timed(name, f):
    def g(*a, **k):
        t = time.perf_counter(); r = f(*a, **k); tm.setdefault(name, []).append(time.perf_counter() - t); return r
    return g
S.solve_values = timed("solve_values", S.solve_values)
S._prepare = timed("prepare", S._prepare)
S._stats = timed("stats", S._stats)
pl = None
for i in range(int(os.environ.get("PROBE_N", "12"))):
    t = time.perf_counter()
    r = solve_batch(mesh, ops, sig, conf)
    tm.setdefault("call", []).append(time.perf_counter() - t)
    tm.setdefault("device", []).append(r.timings["upward"] + r.timings["downward_extract"])
for k, v in tm.items():
    v = np.array(v[2:]) * 1e3
    print(f"{k:14s} median {np.median(v):7.2f} ms  min {v.min():7.2f}  max {v.max():7.2f}  p90 {np.percentile(v, 90):7.2f}")
if "--profile" in sys.argv:
    import cProfile, pstats
    pr = cProfile.Profile()
    pr.enable()
    for i in range(10):
        solve_batch(mesh, ops, sig, conf)
    pr.disable()
    pstats.Stats(pr).sort_stats(sys.argv[-1] if sys.argv[-1] in ("cumulative", "tottime") else "tottime").print_stats(30)
if "--split" in sys.argv:  # host-side time of each step inside solve_values, over PROBE_N calls
    from paper_1104_0623_b200 import plan as PL
    tm.clear()
    PL.Plan.replay_or_run = timed("replay_or_run", PL.Plan.replay_or_run)
    PL.Plan.check_status = timed("check_status", PL.Plan.check_status)
    PL.Plan.workspace = timed("workspace", PL.Plan.workspace)
    torch.cuda.mem_get_info = timed("mem_get_info", torch.cuda.mem_get_info)
    for i in range(int(os.environ.get("PROBE_N", "12"))):
        t = time.perf_counter()
        solve_batch(mesh, ops, sig, conf)
        tm.setdefault("call", []).append(time.perf_counter() - t)
    for k, v in tm.items():
        v = np.array(v) * 1e3
        print(f"split {k:14s} median {np.median(v):7.2f} ms  max {v.max():7.2f}  p90 {np.percentile(v, 90):7.2f}  n {v.size}")
