"""Full-size reference outputs for the BASELINE configs (run in the build container
only; /root/reference does not exist on the GPU box).

    python tests/golden/make_fullscale.py job cfg1 3      # one energy point -> /tmp/fullscale/cfg1_3.npz
    python tests/golden/make_fullscale.py jobs             # list every job (for xargs -P)
    python tests/golden/make_fullscale.py combine          # /tmp/fullscale/* -> tests/golden/full_cfg*.npz

What each fixture holds (every entry of diag(G^r) and diag(G^<), complex128):

* cfg1 (130x130, 16 energies): the reference ``solve`` (solver.py:586-701,
  SolverConfig(kernel='naive', compute_gless=True)) on every energy point.
* cfg2 (256x256 9-point, 64 energies): the reference ``solve`` on energies
  0, 21, 42, 63 (~10-25 min each on one core).
* cfg3 (256x1024, 32 energies): the reference FIND cannot finish at this size
  (set construction is O(n * #clusters)); the reference's own RGF
  (rgf.py:121-136 rgf_gr_diag, rgf.py:178-208 rgf_gless_diag, validated against
  FIND and dense inversion in pkg/tests/test_rgf.py:48-87) on energies 0 and 31.
* cfg4 is not generated here: the reference RGF needs ~120 GB of host RAM and the
  reference FIND cannot build its sets; see ``oracle/fullscale_cfg4.py``.

The inputs are the canonical seeded generator (paper_1104_0623_b200/configs.py,
BASELINE.md §3); the fixtures store only the energy indices and outputs.
"""

import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
OUT = Path(os.environ.get("FULLSCALE_TMP", "/tmp/fullscale"))
sys.path.insert(0, str(HERE.parent.parent))
sys.path.insert(0, "/root/reference/pkg/src")

PLAN = {
    "cfg1": (1, list(range(16)), "find"),
    "cfg2": (2, [0, 21, 42, 63], "find"),
    "cfg3": (3, [0, 31], "rgf"),
}


def run_job(name, k):
    import find_selinv as ref
    from find_selinv.operators import SparseOperator

    from paper_1104_0623_b200.configs import CONFIGS, config_problem

    idx, _, how = PLAN[name]
    cfg = CONFIGS[idx]
    p = config_problem(idx)
    mesh = ref.Mesh(cfg.nx, cfg.ny)
    a_op = SparseOperator(p.a_csr(k))
    s_op = SparseOperator(p.sigma_csr())
    t0 = time.time()
    if how == "find":
        r = ref.solve(mesh, a_op, s_op, ref.SolverConfig(kernel="naive", compute_gless=True))
        gr, gl = r.gr_diag, r.gless_diag
        w = r.ledger.multiplications
        wnum, wden = w.numerator, w.denominator
    else:
        from find_selinv.rgf import block_partition, rgf_gless_diag, rgf_gr_diag

        bt = block_partition(a_op, mesh)
        gr = rgf_gr_diag(bt)
        sbt = block_partition(s_op, mesh)
        gl = rgf_gless_diag(bt, sbt)
        wnum, wden = 0, 1
    dt = time.time() - t0
    OUT.mkdir(parents=True, exist_ok=True)
    np.savez(OUT / f"{name}_{k}.npz", gr=gr, gl=gl, seconds=dt, wnum=str(wnum), wden=str(wden))
    print(name, k, how, f"{dt:.1f} s", flush=True)


def combine():
    for name, (idx, ks, how) in PLAN.items():
        files = [OUT / f"{name}_{k}.npz" for k in ks]
        if not all(f.exists() for f in files):
            print("incomplete", name, [f.name for f in files if not f.exists()])
            continue
        d = [np.load(f) for f in files]
        src = ("reference solve (solver.py:586), SolverConfig(kernel='naive', compute_gless=True)" if how == "find"
               else "reference RGF (rgf.py:121-136 rgf_gr_diag, rgf.py:178-208 rgf_gless_diag)")
        np.savez(HERE / f"full_{name}.npz", config=idx, energy_idx=np.array(ks), gr=np.array([x["gr"] for x in d]),
                 gl=np.array([x["gl"] for x in d]), seconds=np.array([float(x["seconds"]) for x in d]), source=src)
        print("wrote", name, [float(x["seconds"]) for x in d])


if __name__ == "__main__":
    if sys.argv[1] == "job":
        run_job(sys.argv[2], int(sys.argv[3]))
    elif sys.argv[1] == "jobs":
        # longest first so the pool drains evenly
        order = [("cfg2", k) for k in PLAN["cfg2"][1]] + [("cfg3", k) for k in PLAN["cfg3"][1]] + \
                [("cfg1", k) for k in PLAN["cfg1"][1]]
        for n, k in order:
            print(n, k)
    elif sys.argv[1] == "combine":
        combine()
