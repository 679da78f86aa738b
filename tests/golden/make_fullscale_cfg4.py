"""cfg4 (1024x1024, 8 energies) full-size fixture from the pinned CPU oracle port (run in the
build container; needs ~12 GB of host RAM and ~30 min on 8 cores).

    python tests/golden/make_fullscale_cfg4.py [energy_index ...]     # default: 0

Why the port and not the reference: at 1024x1024 the reference FIND cannot build its sets
(mesh.py:209-232 is O(n * #clusters): hours), and the reference RGF holds all 2 x 1024 dense
1024 x 1024 connected blocks (rgf.py:108-208; about 120 GB of host RAM, this container has 62 GB).
oracle/find_oracle.py restates the reference path with the same LAPACK calls per elimination; it
is pinned to the reference's own outputs on every full-size fixture the reference can produce
(tests/test_oracle_golden.py: cfg0-cfg2 FIND, cfg3 RGF), so its cfg4 output stands in for the
reference there.  tests/test_fullscale.py compares the GPU path against every 8th node (the committed
subset).
"""

import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))

from oracle.find_oracle import FindOracle  # noqa: E402
from paper_1104_0623_b200.configs import config_problem  # noqa: E402


STRIDE = 8


def main(ks):
    p = config_problem(4)
    t0 = time.time()
    o = FindOracle(p.nx, p.ny, p.a_csr(0))
    print("oracle plan", round(time.time() - t0, 1), "s", flush=True)
    gr, gl, secs = [], [], []
    for k in ks:
        t1 = time.time()
        r = o.solve(p.a_csr(k), p.sigma_csr())
        secs.append(time.time() - t1)
        gr.append(r.gr_diag)
        gl.append(r.gless_diag)
        print("energy", k, round(secs[-1], 1), "s", flush=True)
    gr, gl = np.array(gr), np.array(gl)
    # the committed fixture keeps every STRIDE-th node (1 048 576 nodes x 2 vectors x 16 B = 32 MB per energy
    # otherwise) plus the vectors' maxima; the full vectors go to /tmp for the generating session
    np.savez("/tmp/full_cfg4_all.npz", energy_idx=np.array(ks), gr=gr, gl=gl)
    idx = np.arange(0, gr.shape[1], STRIDE)
    np.savez_compressed(HERE / "full_cfg4.npz", config=4, energy_idx=np.array(ks), node_idx=idx, gr=gr[:, idx],
                        gl=gl[:, idx], gr_max=np.abs(gr).max(axis=1), gl_max=np.abs(gl).max(axis=1),
                        seconds=np.array(secs),
                        source="oracle port (oracle/find_oracle.py FindOracle.solve, naive, compute_gless)")
    print("wrote full_cfg4.npz", flush=True)


if __name__ == "__main__":
    main([int(x) for x in sys.argv[1:]] or [0])
