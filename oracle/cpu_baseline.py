"""CPU BASELINE — test/bench infrastructure only (bench.py's cpu_baseline leg and
``--impl reference`` arm).  Never part of the product path.

Times the oracle port of the reference FIND path (oracle/find_oracle.py, which
restates solver.py:188-243 / 392-418 and kernels.py:363-392 with the same
scipy LAPACK calls per elimination) on a BOUNDED, stratified sample of one
energy point's eliminations and extrapolates to the full energy point:

    t_energy = sum over (pass, level) groups of  count_g * mean(t_sampled_g)

Each sampled elimination runs the port's real code (merge gathers from the real
A and Sigma^<, LU with partial pivoting, the two triangular solves, the Schur
and Sigma products, the sorted store); only the child U/R blocks it consumes
are synthetic (well-conditioned, correct shapes), because computing them would
require the whole pass.  LAPACK/BLAS cost does not depend on the values.
"""

from __future__ import annotations

import os
import time

import numpy as np

from .find_oracle import FindOracle, OLedger


def _blk(rng, m):
    if m == 0:
        return np.zeros((0, 0), np.complex128)
    return (4.0 + m) * np.eye(m) + 0.1 * (rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m)))


def elimination_jobs(o: FindOracle):
    """Every elimination of one energy point, grouped by (pass, level)."""
    jobs = {}
    for c in o.bottom_up:
        if c.parent is None:
            continue
        if c.is_leaf:
            order = np.concatenate([c.private_inner, c.boundary])
            jobs.setdefault(("up", c.level), []).append(("seed", c, order))
        else:
            jobs.setdefault(("up", c.level), []).append(("merge", c, None))
    for c in o.by_label.values():
        if c.parent is not None:
            jobs.setdefault(("down", c.level), []).append(("down", c, None))
        if c.is_leaf:
            jobs.setdefault(("final", c.level), []).append(("final", c, None))
    return jobs


def estimate_seconds_per_energy(o: FindOracle, a, sg, fraction=0.125, min_per_group=2, seed=0):
    """Stratified estimate of the port's wall time for one energy point."""
    rng = np.random.default_rng(seed)
    a = a.tocsr()
    sg = sg.tocsr()
    led = OLedger()
    empty = np.array([], np.int64)
    z = np.zeros((0, 0), np.complex128)
    total = 0.0
    timed = 0
    n_all = 0
    t_wall0 = time.perf_counter()
    for key, lst in sorted(elimination_jobs(o).items(), key=lambda kv: (kv[0][0], kv[0][1])):
        n_all += len(lst)
        k = max(min_per_group, int(np.ceil(len(lst) * fraction)))
        idx = np.unique(np.linspace(0, len(lst) - 1, min(k, len(lst))).round().astype(int))
        acc = 0.0
        for i in idx:
            kind, c, order = lst[i]
            if kind == "seed":
                from .find_oracle import extract

                t0 = time.perf_counter()
                sa = extract(a, order, order)
                ss = extract(sg, order, order)
                o._eliminate(a, sg, order, empty, sa, z, ss, z, c.private_inner, c.label, True, led, 1e-12)
                acc += time.perf_counter() - t0
            elif kind == "merge":
                l, r = c.children
                ul, ur = _blk(rng, l.boundary.size), _blk(rng, r.boundary.size)
                rl, rr = _blk(rng, l.boundary.size), _blk(rng, r.boundary.size)
                t0 = time.perf_counter()
                o._eliminate(a, sg, l.boundary, r.boundary, ul, ur, rl, rr, c.private_inner, c.label, True, led, 1e-12)
                acc += time.perf_counter() - t0
            elif kind == "down":
                p = c.parent
                a0, a1 = p.children
                sib = a1 if a0 is c else a0
                left = o.comps[-p.label][0]
                b_set, s_set = o.comps[-c.label]
                pu, pr = _blk(rng, left.size), _blk(rng, left.size)
                su, sr = _blk(rng, sib.boundary.size), _blk(rng, sib.boundary.size)
                t0 = time.perf_counter()
                o._eliminate(a, sg, left, sib.boundary, pu, su, pr, sr, s_set, -c.label, True, led, 1e-12)
                acc += time.perf_counter() - t0
            else:
                ring = o.comps[-c.label][0]
                neg = (_blk(rng, ring.size), _blk(rng, ring.size))
                gr = np.zeros(o.n, np.complex128)
                gl = np.zeros(o.n, np.complex128)
                filled = np.zeros(o.n, bool)
                t0 = time.perf_counter()
                o._leaf(c, a, sg, neg, gr, gl, filled, led, True, 1e-12)
                acc += time.perf_counter() - t0
        timed += len(idx)
        total += acc / len(idx) * len(lst)
    return {
        "seconds_per_energy": total,
        "sampled_eliminations": int(timed),
        "total_eliminations": int(n_all),
        "sample_wall_seconds": time.perf_counter() - t_wall0,
    }


def blas_threads() -> int:
    try:
        from threadpoolctl import threadpool_info

        info = threadpool_info()
        return max([int(i.get("num_threads", 1)) for i in info] or [os.cpu_count() or 1])
    except Exception:
        return os.cpu_count() or 1


def _energy_worker(nx, ny, a, sg, fraction, seed, barrier, out):
    from threadpoolctl import threadpool_limits

    with threadpool_limits(1):
        o = FindOracle(nx, ny, a)
        barrier.wait()
        out.put(estimate_seconds_per_energy(o, a, sg, fraction=fraction, seed=seed))


def parallel_energy_rate(nx, ny, a, sg, workers=None, fraction=0.125, seed=0):
    """Energy-parallel CPU throughput: ``workers`` processes (default: every host core), one BLAS
    thread each, each estimating a different energy point concurrently (all cores busy while every
    sample is timed).  Energy points are independent, so this is how a host sweep uses its cores;
    single-process threaded LAPACK on these block sizes is several times slower (bench.py notes)."""
    import multiprocessing as mp

    workers = workers or os.cpu_count() or 1
    ctx = mp.get_context("spawn")
    keys = ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")
    saved = {k: os.environ.get(k) for k in keys}
    for k in keys:
        os.environ[k] = "1"
    try:
        barrier, out = ctx.Barrier(workers), ctx.Queue()
        procs = [ctx.Process(target=_energy_worker, args=(nx, ny, a, sg, fraction, seed + w, barrier, out))
                 for w in range(workers)]
        for p in procs:
            p.start()
        res = [out.get() for _ in procs]
        for p in procs:
            p.join()
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    t = [r["seconds_per_energy"] for r in res]
    return {
        "rate": float(sum(1.0 / x for x in t)),
        "seconds_per_energy": float(np.mean(t)),
        "workers": workers,
        "sampled_eliminations": res[0]["sampled_eliminations"],
        "total_eliminations": res[0]["total_eliminations"],
        "sample_wall_seconds": float(max(r["sample_wall_seconds"] for r in res)),
    }
