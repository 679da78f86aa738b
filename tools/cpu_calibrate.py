"""Calibrate the sampled CPU-baseline estimator (oracle/cpu_baseline.py) against a full,
unsampled run of the same oracle port on one cfg1 energy point (both on one core, one BLAS
thread).  Writes profiles/r02_cpu_calibration.json.

    OPENBLAS_NUM_THREADS=1 python tools/cpu_calibrate.py
"""
import json
import os
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import numpy as np  # noqa: E402

from oracle.cpu_baseline import buckets_of, elimination_jobs, estimate_step  # noqa: E402
from oracle.find_oracle import FindOracle  # noqa: E402
from paper_1104_0623_b200.configs import config_problem  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
p = config_problem(cfg, 1)
a, sg = p.a_csr(0).tocsr(), p.sigma_csr().tocsr()
o = FindOracle(p.nx, p.ny, a)
t0 = time.perf_counter()
o.solve(a, sg)
full = time.perf_counter() - t0
b = buckets_of(elimination_jobs(o))
rng = np.random.default_rng(0)
est = [estimate_step(o, b, a, sg, rng)["seconds_per_energy"] for _ in range(8)]
out = {"config": cfg, "full_run_seconds": full, "estimates_seconds": est, "estimate_mean": float(np.mean(est)),
       "estimate_over_full": float(np.mean(est) / full), "estimate_cv": float(np.std(est) / np.mean(est)),
       "note": "one process, one BLAS thread; the estimator's per-step sample is one random elimination per "
               "(kind, s, b) bucket (oracle/cpu_baseline.py)"}
print(json.dumps(out))
(ROOT / "profiles" / f"r02_cpu_calibration_cfg{cfg}.json").write_text(json.dumps(out, indent=1))
