"""CPU BASELINE — test/bench infrastructure only (bench.py's cpu_baseline leg and
``--impl reference`` arm).  Never part of the product path.

Times the oracle port of the reference FIND path (oracle/find_oracle.py, which
restates solver.py:188-243 / 392-418 and kernels.py:363-392 with the same
scipy LAPACK calls per elimination) on a BOUNDED sample of one energy point's
eliminations and extrapolates to the full energy point.

Estimator (one "step"):

* every elimination of the energy point (upward seeds and merges, downward
  complement merges, final leaf steps) is put in a bucket keyed by (kind,
  half-octave of s, half-octave of b);
* in every bucket, one randomly chosen member whose reference work W
  (kernels.py:90-91 naive counts, complex mults) is at most ``cap`` is run for
  real and timed; the bucket's members up to ``cap`` are charged count x that
  time;
* members above ``cap`` (the large dense separators: their time is LAPACK/BLAS
  bound) are charged W / rate, where rate is the complex mults per second the
  timed eliminations of this step reached (those with W >= 1e7, i.e. the
  BLAS-bound ones).

Each sampled elimination runs the port's real code (merge gathers from the
real A(E_k) and Sigma^<, LU with partial pivoting, the two triangular solves,
the Schur and Sigma products, the sorted store); only the child U/R blocks it
consumes are synthetic (well-conditioned, correct shapes), because computing
them would require the whole pass.  LAPACK/BLAS cost does not depend on the
values.

Energy-parallel: ``workers`` forked processes (one per host core, one BLAS
thread each), worker w on energy point w mod nE, all timing their samples
concurrently (a barrier per step); throughput = sum of the per-process rates.

    python -m oracle.cpu_baseline --config 4 --steps 1 --warmup 0      # one JSON line
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

for _k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_k, "1")

import numpy as np  # noqa: E402

from .find_oracle import FindOracle, OLedger, extract, naive_dense_count, sigma_naive_count  # noqa: E402

CAP = 3e8          # complex mults: members above are charged by the measured BLAS rate
RATE_MIN_W = 1e7   # timed eliminations at least this large define that rate


def _blk(rng, m):
    if m == 0:
        return np.zeros((0, 0), np.complex128)
    return (4.0 + m) * np.eye(m) + 0.1 * (rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m)))


def _w(s, b, leaf_c=0):
    w = float(naive_dense_count(s, b) + sigma_naive_count(s, b)) if s else 0.0
    return w + 3.0 * leaf_c ** 3  # dense inverse + G^< sandwich of a final step (solver.py:388, 664)


def _hbin(x):
    return 0 if x <= 0 else int(np.ceil(2 * np.log2(x + 1)))


def elimination_jobs(o: FindOracle):
    """Every elimination of one energy point: (kind, cluster, s, b, W)."""
    jobs = []
    for c in o.bottom_up:
        if c.parent is None:
            continue
        s, b = c.private_inner.size, c.boundary.size
        jobs.append(("seed" if c.is_leaf else "merge", c, s, b, _w(s, b)))
    for c in o.by_label.values():
        if c.parent is not None:
            b_set, s_set = o.comps[-c.label]
            jobs.append(("down", c, s_set.size, b_set.size, _w(s_set.size, b_set.size)))
        if c.is_leaf:
            ring = o.comps[-c.label][0]
            jobs.append(("final", c, ring.size, c.nodes.size, _w(ring.size, c.nodes.size, c.nodes.size)))
    return jobs


def buckets_of(jobs):
    out = {}
    for j in jobs:
        out.setdefault((j[0], _hbin(j[2]), _hbin(j[3])), []).append(j)
    return out


def run_job(o: FindOracle, job, a, sg, rng, led):
    """Run one elimination of the port for real; returns its wall time (s)."""
    kind, c = job[0], job[1]
    empty = np.array([], np.int64)
    z = np.zeros((0, 0), np.complex128)
    if kind == "seed":
        t0 = time.perf_counter()
        order = np.concatenate([c.private_inner, c.boundary])
        sa = extract(a, order, order)
        ss = extract(sg, order, order)
        o._eliminate(a, sg, order, empty, sa, z, ss, z, c.private_inner, c.label, True, led, 1e-12)
        return time.perf_counter() - t0
    if kind == "merge":
        l, r = c.children
        ul, ur = _blk(rng, l.boundary.size), _blk(rng, r.boundary.size)
        rl, rr = _blk(rng, l.boundary.size), _blk(rng, r.boundary.size)
        t0 = time.perf_counter()
        o._eliminate(a, sg, l.boundary, r.boundary, ul, ur, rl, rr, c.private_inner, c.label, True, led, 1e-12)
        return time.perf_counter() - t0
    if kind == "down":
        p = c.parent
        a0, a1 = p.children
        sib = a1 if a0 is c else a0
        left = o.comps[-p.label][0]
        s_set = o.comps[-c.label][1]
        pu, pr = _blk(rng, left.size), _blk(rng, left.size)
        su, sr = _blk(rng, sib.boundary.size), _blk(rng, sib.boundary.size)
        t0 = time.perf_counter()
        o._eliminate(a, sg, left, sib.boundary, pu, su, pr, sr, s_set, -c.label, True, led, 1e-12)
        return time.perf_counter() - t0
    ring = o.comps[-c.label][0]
    neg = (_blk(rng, ring.size), _blk(rng, ring.size))
    gr = np.zeros(o.n, np.complex128)
    gl = np.zeros(o.n, np.complex128)
    filled = np.zeros(o.n, bool)
    t0 = time.perf_counter()
    o._leaf(c, a, sg, neg, gr, gl, filled, led, True, 1e-12)
    return time.perf_counter() - t0


def estimate_step(o: FindOracle, buckets, a, sg, rng, cap=CAP):
    """One sampled estimate of the port's wall time for one energy point (seconds)."""
    led = OLedger()
    t_small = 0.0
    w_large = 0.0
    rate_w = rate_t = 0.0
    timed = 0
    t_wall0 = time.perf_counter()
    for key in sorted(buckets):
        lst = buckets[key]
        small = [j for j in lst if j[4] <= cap]
        w_large += sum(j[4] for j in lst if j[4] > cap)
        if not small:
            continue
        j = small[int(rng.integers(len(small)))]
        t = run_job(o, j, a, sg, rng, led)
        timed += 1
        t_small += t * len(small)
        if j[4] >= RATE_MIN_W:
            rate_w += j[4]
            rate_t += t
    if w_large and rate_t == 0.0:  # no BLAS-bound member was drawn: time the largest one below the cap
        j = max((j for lst in buckets.values() for j in lst if j[4] <= cap), key=lambda q: q[4])
        rate_t = run_job(o, j, a, sg, rng, led)
        rate_w = j[4]
        timed += 1
    rate = rate_w / rate_t if rate_t else 0.0
    t_large = w_large / rate if w_large else 0.0
    return {"seconds_per_energy": t_small + t_large, "timed_seconds_part": t_small, "rate_part_seconds": t_large,
            "blas_rate_cmults_per_s": rate, "sampled_eliminations": timed,
            "sample_wall_seconds": time.perf_counter() - t_wall0}


# ---------------------------------------------------------------------------- energy-parallel driver

_STATE: dict = {}


def _worker(w, steps, seed, barrier, out):
    from threadpoolctl import threadpool_limits

    o, p, buckets = _STATE["o"], _STATE["p"], _STATE["buckets"]
    k = w % p.energies.size
    a = p.a_csr(k).tocsr()
    sg = p.sigma_csr().tocsr()
    rng = np.random.default_rng(seed + 7919 * w)
    with threadpool_limits(1):
        for step in range(steps):
            barrier.wait()
            r = estimate_step(o, buckets, a, sg, rng)
            r["worker"], r["step"], r["energy"] = w, step, k
            out.put(r)


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def energy_parallel(cfg_index: int, steps: int = 1, warmup: int = 0, workers: int | None = None, seed: int = 0,
                    problem=None):
    """Returns per-step rates (energy points/s, sum over workers) and metadata."""
    import multiprocessing as mp

    from paper_1104_0623_b200.configs import config_problem

    t0 = time.perf_counter()
    p = problem if problem is not None else config_problem(cfg_index)
    o = FindOracle(p.nx, p.ny, p.a_csr(0))
    jobs = elimination_jobs(o)
    buckets = buckets_of(jobs)
    setup = time.perf_counter() - t0
    _STATE.update(o=o, p=p, buckets=buckets)
    workers = workers or host_cores()
    ctx = mp.get_context("fork")  # the oracle's sets are shared copy-on-write
    total = warmup + steps
    barrier, out = ctx.Barrier(workers), ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(w, total, seed, barrier, out)) for w in range(workers)]
    for pr in procs:
        pr.start()
    res = [out.get() for _ in range(workers * total)]
    for pr in procs:
        pr.join()
    _STATE.clear()
    per_step = []
    for step in range(warmup, total):
        rs = [r for r in res if r["step"] == step]
        per_step.append({"rate": float(sum(1.0 / r["seconds_per_energy"] for r in rs)),
                         "seconds_per_energy": float(np.mean([r["seconds_per_energy"] for r in rs])),
                         "rate_part_share": float(np.mean([r["rate_part_seconds"] / r["seconds_per_energy"]
                                                           for r in rs])),
                         "blas_gflops": float(np.mean([8e-9 * r["blas_rate_cmults_per_s"] for r in rs])),
                         "sampled": int(np.mean([r["sampled_eliminations"] for r in rs])),
                         "wall": float(max(r["sample_wall_seconds"] for r in rs))})
    return {"config": cfg_index, "workers": workers, "setup_seconds": setup, "eliminations": len(jobs),
            "buckets": len(buckets), "cap_cmults": CAP, "steps": per_step}


def describe(r) -> str:
    st = r["steps"]
    return (f"oracle port of reference solve (naive, compute_gless) on cfg{r['config']}, energy-parallel: "
            f"{r['workers']} forked processes x 1 BLAS thread, worker w on energy point w mod nE, timed concurrently; "
            f"per process and step one random real elimination per (kind, s, b) bucket "
            f"({st[0]['sampled']} of {r['eliminations']}, {r['buckets']} buckets) charged x bucket count, "
            f"members above {r['cap_cmults']:.0e} complex mults charged at the timed BLAS rate "
            f"({st[0]['blas_gflops']:.1f} GFLOP/s per core; {100 * st[0]['rate_part_share']:.0f} % of the estimate); "
            f"{np.mean([s['seconds_per_energy'] for s in st]):.1f} s per energy point per process; value = sum of "
            f"per-process rates")


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=0)
    ap.add_argument("--workers", type=int, default=0)
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args(argv)
    r = energy_parallel(args.config, args.steps, args.warmup, args.workers or None, args.seed)
    r["sample"] = describe(r)
    print(json.dumps(r), flush=True)


if __name__ == "__main__":
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    main()
