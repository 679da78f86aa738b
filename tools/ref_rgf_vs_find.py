"""Error level of the problem itself (build container only: imports the reference read-only).

The reference's own two algorithms, FIND (tests/golden/full_cfg1.npz, solver.py:586) and RGF
(rgf.py:121-208), are compared entry by entry on every cfg1 energy point; their disagreement is
the conditioning floor (eps * kappa(A(E)) with eta = 1e-6 in-band energies) any third algorithm,
such as the GPU path, can be expected to reach.  Writes profiles/r02_ref_rgf_vs_find_cfg1.json.
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
from find_selinv import Mesh  # noqa: E402
from find_selinv.operators import SparseOperator  # noqa: E402
from find_selinv.rgf import block_partition, rgf_gless_diag, rgf_gr_diag  # noqa: E402

from paper_1104_0623_b200.configs import config_problem  # noqa: E402

f = np.load(ROOT / "tests" / "golden" / "full_cfg1.npz")
p = config_problem(1)
mesh = Mesh(p.nx, p.ny)
out = []
for i, k in enumerate(f["energy_idx"]):
    a = SparseOperator(p.a_csr(int(k)))
    s = SparseOperator(p.sigma_csr())
    bt = block_partition(a, mesh)
    gr = rgf_gr_diag(bt)
    gl = rgf_gless_diag(bt, block_partition(s, mesh))
    out.append({"energy": int(k), "gr": float(np.abs(gr - f["gr"][i]).max() / np.abs(f["gr"][i]).max()),
                "gl": float(np.abs(gl - f["gl"][i]).max() / np.abs(f["gl"][i]).max())})
    print(out[-1], flush=True)
(ROOT / "profiles" / "r02_ref_rgf_vs_find_cfg1.json").write_text(json.dumps(
    {"what": "reference RGF vs reference FIND, max|d|/max|ref| per cfg1 energy point", "rows": out}, indent=1))
