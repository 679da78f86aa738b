"""CTA-path variants (panel widths and kinds, tile engines, one-CTA tall panels, dependency
scheduling, wide blocks, per-tile inverses) against the
reference's golden outputs, each selected through its environment switch in a fresh
process (the choices are read once per process / plan)."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

SCRIPT = r"""
import json, sys
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import numpy as np
from conftest import load_golden, problem_from_golden, stencil_ops
from paper_1104_0623_b200 import Mesh, SolverConfig, SparseOperator, solve, solve_batch
out = {{}}
for name in ("cfg0", "c5_16x12", "c9_20x20", "c5_8x30"):
    g = load_golden(name); p = problem_from_golden(g)
    ops = [SparseOperator(p.a_csr(k)) for k in range(p.energies.size)]
    r = solve_batch(Mesh(p.nx, p.ny), ops, SparseOperator(p.sigma_csr()), SolverConfig())
    out[name] = [float(np.max(np.abs(r.gr_diag - g["gr"])) / np.max(np.abs(g["gr"]))),
                 float(np.max(np.abs(r.gless_diag - g["gl"])) / np.max(np.abs(g["gl"])))]
for name in ("stencil_16x16", "stencil_8x8"):
    g = load_golden(name); mesh, a, s = stencil_ops(g)
    r = solve(mesh, a, s, SolverConfig(leaf_max=2))
    out[name] = [float(np.max(np.abs(r.gr_diag - g["gr_2"])) / np.max(np.abs(g["gr_2"]))),
                 float(np.max(np.abs(r.gless_diag - g["gl_2"])) / np.max(np.abs(g["gl_2"])))]
print("RESULT", json.dumps(out))
"""


@pytest.mark.parametrize("env", [{}, {"FIND_B200_NB": "16"}, {"FIND_B200_NB": "8"}, {"FIND_B200_SMEM_PANEL": "1"},
                                 {"FIND_B200_TMA": "0"}, {"FIND_B200_TMA_MIN_S": "0"}, {"FIND_B200_CSTAGE": "1"},
                                 {"FIND_B200_TALL_MIN_PANELS": "0", "FIND_B200_TALL_MIN_ROWS": "32"},
                                 {"FIND_B200_DAG_MAX_N": "100000"}, {"FIND_B200_WIDE_MIN_S": "0"},
                                 {"FIND_B200_INV_LAUNCH": "0"}, {"FIND_B200_STRUCT": "0"},
                                 {"FIND_B200_SPLIT_K": "1"}, {"FIND_B200_SPLIT_K": "3"}])
def test_cta_path_variants_match_golden(cuda, env):
    code = SCRIPT.format(root=str(ROOT), tests=str(ROOT / "tests"))
    r = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [l for l in r.stdout.splitlines() if l.startswith("RESULT")][-1]
    res = json.loads(line[len("RESULT "):])
    for name, (egr, egl) in res.items():
        assert egr < 1e-10 and egl < 1e-10, (name, egr, egl, env)



HASH_SCRIPT = r"""
import hashlib, sys
sys.path.insert(0, {root!r})
from paper_1104_0623_b200.configs import build_problem
from paper_1104_0623_b200.plan import plan_for
from paper_1104_0623_b200.solver import sigma_symmetry, solve_values
p = build_problem(96, 40, [0.9, 2.7], seed=17, stencil=5)
plan, _ = plan_for(p.nx, p.ny, p.indptr, p.indices)
gr, gl, _, _ = solve_values(plan, p.a_vals_all(), p.s_vals, sigma_sym=sigma_symmetry(p.sigma_csr()))
print("HASH", hashlib.sha1(gr.tobytes() + gl.tobytes()).hexdigest())
"""


def test_structural_zero_skips_are_bit_identical(cuda):
    """The skipped (B_r, S_l) products are exact zeros: results bit-identical with and without."""
    code = HASH_SCRIPT.format(root=str(ROOT))
    out = []
    for v in ("1", "0"):
        r = subprocess.run([sys.executable, "-c", code], env={**os.environ, "FIND_B200_STRUCT": v},
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        out.append([l for l in r.stdout.splitlines() if l.startswith("HASH")][-1])
    assert out[0] == out[1]


TALL_SCRIPT = r"""
import hashlib, sys
sys.path.insert(0, {root!r})
from paper_1104_0623_b200.configs import build_problem
from paper_1104_0623_b200.plan import plan_for
from paper_1104_0623_b200.solver import sigma_symmetry, solve_values
p = build_problem({nx}, {ny}, [0.9, 2.7], seed=23, stencil=5)
plan, _ = plan_for(p.nx, p.ny, p.indptr, p.indices)
gr, gl, _, _ = solve_values(plan, p.a_vals_all(), p.s_vals, sigma_sym=sigma_symmetry(p.sigma_csr()))
print("HASH", hashlib.sha1(gr.tobytes() + gl.tobytes()).hexdigest())
"""


@pytest.mark.parametrize("nx,ny", [(96, 40), (600, 12), (1030, 6)])
def test_tall_panel_kernel_is_bit_identical(cuda, nx, ny):
    """One-CTA tall panels (1, 2 and 3 rows per thread: dense contact rows of 96 / 600 / 1030 nodes) against
    the register-row CTA / cluster panels: same pivots, same per-element update order, same bits."""
    code = TALL_SCRIPT.format(root=str(ROOT), nx=nx, ny=ny)
    out = []
    for env in ({"FIND_B200_TALL_MIN_PANELS": "0", "FIND_B200_TALL_MIN_ROWS": "32"},
                {"FIND_B200_TALL_MIN_PANELS": "1000000000"}):
        r = subprocess.run([sys.executable, "-c", code], env={**os.environ, **env}, capture_output=True, text=True,
                           timeout=900)
        assert r.returncode == 0, r.stderr[-2000:]
        out.append([l for l in r.stdout.splitlines() if l.startswith("HASH")][-1])
    assert out[0] == out[1]


@pytest.mark.gpu
def test_two_devices_in_one_process():
    """Kernel attributes and side streams are per device: a solve on cuda:0 then on cuda:1 (needs 2 GPUs)."""
    import torch

    if torch.cuda.device_count() < 2:
        pytest.skip("needs two CUDA devices")
    from paper_1104_0623_b200 import Mesh, SolverConfig, SparseOperator, solve
    from paper_1104_0623_b200.configs import build_problem

    p = build_problem(12, 10, [1.2], seed=3)
    out = []
    for d in (0, 1):
        with torch.cuda.device(d):
            r = solve(Mesh(p.nx, p.ny), SparseOperator(p.a_csr(0)), SparseOperator(p.sigma_csr()), SolverConfig())
            out.append(r)
    np.testing.assert_allclose(out[0].gr_diag, out[1].gr_diag, rtol=0, atol=1e-13 * np.abs(out[0].gr_diag).max())
