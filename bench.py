"""Benchmark of the FIND selected-inversion hot path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1] [--impl reference]

Workload (BASELINE.json configs[1]): 130x130 mesh, 5-point stencil with dense
contact self-energies, 16 energy points solved as one batch; outputs
diag(G^r) and diag(G^<) per energy.  One "step" = one selected inversion of
all 16 energy points.  Metric: energy points/s (whole job, all GPUs).

`value`   device throughput, inputs resident in HBM, CUDA events on the solve
          stream, L2 flushed (256 MiB write) between timed steps.
`e2e`     the same metric through the public drop-in API
          (paper_1104_0623_b200.solve_batch on SparseOperator inputs): host
          validation, pinned H2D of the step's A(E_k)/Sigma^< values, kernels,
          D2H of both diagonals; host wall clock per step.
`roofline` the dominant kernel (by device time) against the measured FP64
          tensor peak (DMMA microbenchmark, profiles/r01_fp64_probe.txt); work
          is the reference ledger W (complex mults, kernels.py:88-146) x 8 flop.
`cpu_baseline` the oracle port of the reference path (oracle/), stratified
          sample of one energy point's eliminations, extrapolated (rank 0, N=1).

--impl reference: times the oracle port (the reference's algorithm and LAPACK
calls, oracle/find_oracle.py) on the host cores, same metric/config.
Multi-GPU: replicas (energy sharding, no data-path collective): each rank
solves its own 16 energy points; value = N*16*K / max-over-ranks time.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

FP64_PEAK_TFLOPS = 37.19  # measured: mma.sync m8n8k4 f64 (DMMA.8x8x4), 148 SMs @1965 MHz (profiles/r01_fp64_probe.txt)
ZGEMM_TFLOPS = 37.02      # measured: cuBLAS ZGEMM 8192^3 via torch (profiles/r01_blas_probe.txt)
METRIC = "energy points/sec per mesh (diag G^r + G^<)"
UNIT = "energy points/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--levels", default="", help="write per-launch-group timings (json) to this path")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md)."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None
        self.th = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.th is not None:
            self.th.join(timeout=2)
        sm = []
        smax = None
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                smax = float(r[1])
                for nm, v in zip(names, r[4:8]):
                    if v.strip().lower() == "active":
                        reasons.add(nm)
            except Exception:
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_baseline_line(cfg_index, p, fraction=0.125):
    from oracle.cpu_baseline import parallel_energy_rate

    r = parallel_energy_rate(p.nx, p.ny, p.a_csr(0).tocsr(), p.sigma_csr().tocsr(), fraction=fraction)
    return {
        "value": r["rate"],
        "unit": UNIT,
        "cores": r["workers"],
        "kind": "port",
        "sample": (f"oracle port of reference solve (naive, compute_gless) on cfg{cfg_index}, energy-parallel: "
                   f"{r['workers']} processes x 1 BLAS thread, each a different energy point, concurrently; per "
                   f"process a stratified {r['sampled_eliminations']}/{r['total_eliminations']} elimination sample "
                   f"({r['sample_wall_seconds']:.1f} s wall) extrapolated per (pass, level) group; "
                   f"{r['seconds_per_energy']:.2f} s per energy point per process; value = sum of per-process rates"),
    }


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_1104_0623_b200.configs import CONFIGS, config_problem

    cfg = CONFIGS[args.config]
    p = config_problem(args.config, 1)
    from oracle.cpu_baseline import parallel_energy_rate

    a, sg = p.a_csr(0).tocsr(), p.sigma_csr().tocsr()
    frac = 0.125 if args.config > 0 else 1.0
    for w in range(args.warmup):
        parallel_energy_rate(p.nx, p.ny, a, sg, fraction=min(frac, 0.02), seed=1000 + 100 * w)
    rates, walls, workers = [], [], 1
    for k in range(args.steps):
        r = parallel_energy_rate(p.nx, p.ny, a, sg, fraction=frac, seed=100 * k)
        rates.append(r["rate"])
        walls.append(r["sample_wall_seconds"])
        workers = r["workers"]
    v = float(np.mean(rates))
    t = 1.0 / v
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": f"cfg{args.config}: {cfg.nx}x{cfg.ny} {cfg.stencil}-point, {cfg.n_energies} energy "
                               f"points, diag G^r + G^<", "mesh": [cfg.nx, cfg.ny], "n_energies": cfg.n_energies},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": workers, "kind": "port",
                         "sample": (f"per step: oracle port (reference algorithm, scipy LAPACK per elimination), "
                                    f"energy-parallel: {workers} processes x 1 BLAS thread, each a stratified "
                                    f"{frac:.3f} sample of a different energy point's eliminations, extrapolated; "
                                    f"value = sum of per-process rates; mean sample wall {np.mean(walls):.1f} s")},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_b200(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    from paper_1104_0623_b200 import Mesh, SolverConfig, SparseOperator, solve_batch
    from paper_1104_0623_b200.configs import CONFIGS, config_problem
    from paper_1104_0623_b200.plan import plan_for

    cfg = CONFIGS[args.config]
    p = config_problem(args.config)
    n_e = p.energies.size
    plan, _ = plan_for(p.nx, p.ny, p.indptr, p.indices)
    W = float(plan.native_work(0))
    stream = torch.cuda.Stream(dev)
    a_host = torch.from_numpy(p.a_vals_all()).pin_memory()
    s_host = torch.from_numpy(p.s_vals).pin_memory()
    a_d = a_host.to(dev)
    s_d = s_host.to(dev)
    gr_d = torch.empty((n_e, plan.n), dtype=torch.complex128, device=dev)
    gl_d = torch.empty((n_e, plan.n), dtype=torch.complex128, device=dev)
    ws = plan.workspace(n_e, True, dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()

    from paper_1104_0623_b200.solver import sigma_symmetry

    ssym = sigma_symmetry(p.sigma_csr())

    def step_eager():
        plan.run(a_d, s_d, gr_d, gl_d, ws=ws, stream=stream, sigma_sym=ssym)

    # the timed steps replay the solve's launch schedule as one captured CUDA graph (as the public
    # API does from its second call, Plan.replay_or_run); the instrumented step below runs eagerly
    graph = None

    def step():
        graph.replay() if graph is not None else step_eager()

    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 3) - 1):
            step_eager()
        plan.check_status(ws, n_e, stream)
        if os.environ.get("FIND_B200_GRAPH", "1") != "0":
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream):
                step_eager()
        step()  # last warm-up step (the graph's first replay)
        plan.check_status(ws, n_e, stream)
    # ---- timed region: K steps, L2 flushed between steps (outside the events) ----
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clocks = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    with torch.cuda.stream(stream):
        for k in range(args.steps):
            flush.fill_(k & 0xff)
            evs[k][0].record(stream)
            step()
            evs[k][1].record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    plan.check_status(ws, n_e, stream)
    dev_ms = sum(a.elapsed_time(b) for a, b in evs)
    t_max = torch.tensor([dev_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    dev_ms = float(t_max.item())
    ms_per_step = dev_ms / args.steps
    value = world * n_e * args.steps / (dev_ms * 1e-3)

    # ---- per-launch timing: one extra instrumented step with every launch group run ALONE
    #      (groups in plan order on the solve stream, so each launch's CUDA-event duration is
    #      its own, not shared with concurrent groups) -> per-kind roofline, live
    import ctypes as C

    from paper_1104_0623_b200 import _native
    from paper_1104_0623_b200.workmodel import KINDS, TENSOR_KINDS, executed_cmacs

    lib = _native.lib()
    ngroups = len(plan.groups["count"])
    with torch.cuda.stream(stream):
        flush.fill_(1)
        torch.cuda.synchronize()
        lib.find_solve_timing_enable(1)
        for gi in range(ngroups):
            plan.run(a_d, s_d, gr_d, gl_d, ws=ws, stream=stream, sigma_sym=ssym, groups=(gi, gi + 1))
        torch.cuda.synchronize()
        lib.find_solve_timing_enable(0)
    nl = int(lib.find_solve_timing_read(None, None, None, 0))
    kk = (C.c_int32 * nl)()
    gg = (C.c_int32 * nl)()
    ms = (C.c_float * nl)()
    lib.find_solve_timing_read(kk, gg, ms, nl)
    work = executed_cmacs(plan, ssym)
    per_kind = {}
    per_group_ms = np.zeros(ngroups)
    for i in range(nl):
        name = KINDS[kk[i]]
        d = per_kind.setdefault(name, {"ms": 0.0, "launches": 0, "cmacs": 0.0, "groups": set()})
        d["ms"] += ms[i]
        d["launches"] += 1
        d["groups"].add(gg[i])
        per_group_ms[gg[i]] += ms[i]
    for name, d in per_kind.items():
        d["cmacs"] = sum(work.get((gi, name), 0.0) for gi in d["groups"]) * n_e
    tot_ms = sum(d["ms"] for d in per_kind.values())

    def kind_line(d):
        tf = 8 * d["cmacs"] / (d["ms"] * 1e-3) / 1e12 if d["cmacs"] and d["ms"] else None
        return {"ms_per_step_serialized": round(d["ms"], 3), "share": round(d["ms"] / tot_ms, 4),
                "launches": d["launches"], "tflops": round(tf, 3) if tf else None,
                "frac_fp64_peak": round(tf / FP64_PEAK_TFLOPS, 4) if tf else None}

    kernels = {name: kind_line(d) for name, d in sorted(per_kind.items(), key=lambda kv: -kv[1]["ms"])}
    dom = max((k for k in per_kind if k in TENSOR_KINDS), key=lambda k: per_kind[k]["ms"])
    dk = per_kind[dom]
    achieved = 8 * dk["cmacs"] / (dk["ms"] * 1e-3) / 1e12
    traffic = None
    prof = ROOT / "profiles" / "r01_ncu_kernels.json"
    if prof.exists():
        traffic = json.loads(prof.read_text()).get(f"{dom}_kernel", {}).get("dram_bytes_per_launch")
    roofline = {
        "bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
        "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
        "kernel": f"{dom}_kernel", "launches_per_step": dk["launches"], "share_of_step": dk["ms"] / tot_ms,
        "peak_source": "measured FP64 DMMA microbenchmark (profiles/r01_fp64_probe.txt); cuBLAS ZGEMM 37.02",
        "work": "executed complex MACs x 8 of those launches (paper_1104_0623_b200/workmodel.py) / their CUDA-event "
                "durations with each launch group run alone (serialized instrumented step); dominant = the FP64 "
                "tensor-core (DMMA) kind with the largest serialized device time; traffic = ncu dram bytes per launch "
                "of that kernel (profiles/r01_ncu_kernels.json)",
    }
    # north-star target: FP64 fraction on the near-root levels (upward levels 1-4, downward 1-4)
    g = plan.groups
    wl = {}
    for (gi, kname), v in work.items():
        wl[gi] = wl.get(gi, 0.0) + v
    near = [gi for gi in range(ngroups) if int(g["level"][gi]) <= 4 and int(g["pass"][gi]) in (0, 1)]
    near_ms = float(per_group_ms[near].sum())
    near_tf = 8 * sum(wl.get(gi, 0.0) for gi in near) * n_e / (near_ms * 1e-3) / 1e12 if near_ms else 0.0
    near_root = {"levels": "upward 1-4 + downward 1-4", "groups": len(near), "ms_serialized": round(near_ms, 3),
                 "tflops": round(near_tf, 3), "frac_fp64_peak": round(near_tf / FP64_PEAK_TFLOPS, 4)}
    if args.levels and rank == 0:
        Path(args.levels).write_text(json.dumps({"kernels": kernels, "launches": [
            {"kind": KINDS[kk[i]], "group": int(gg[i]), "ms": float(ms[i])} for i in range(nl)]}, indent=1))

    # ---- e2e through the public API (host SparseOperators -> diagonals on host) ----
    mesh = Mesh(p.nx, p.ny)
    ops = [SparseOperator(p.a_csr(k)) for k in range(n_e)]
    sig = SparseOperator(p.sigma_csr())
    conf = SolverConfig()
    # 20 calls, median: the host side sees sporadic 30-100 ms stalls from the box (bursts of a
    # few calls, with or without Python's GC) while the device time per call stays flat
    e2e_steps = 20
    per_step = []
    parts = []
    with torch.cuda.stream(stream):
        solve_batch(mesh, ops, sig, conf)  # eager
        solve_batch(mesh, ops, sig, conf)  # captures the level schedule as CUDA graphs
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        for _ in range(e2e_steps):
            t0 = time.perf_counter()
            res = solve_batch(mesh, ops, sig, conf)  # returns host arrays: D2H + sync inside
            per_step.append(time.perf_counter() - t0)
            parts.append((res.timings["tree"], res.timings["upward"] + res.timings["downward_extract"],
                          res.timings["total"]))
    e2e_s = float(np.median(per_step))
    t_e = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_e, op=dist.ReduceOp.MAX)
    e2e_s = float(t_e.item())
    e2e = {"value": world * n_e / e2e_s, "unit": UNIT, "steps": e2e_steps,
           "timing": "host wall clock per solve_batch call, median over the steps (max over ranks)",
           "median_host_prepare_ms": round(1e3 * float(np.median([x[0] for x in parts])), 3),
           "median_device_ms": round(1e3 * float(np.median([x[1] for x in parts])), 3),
           "median_call_ms": round(1e3 * float(np.median([x[2] for x in parts])), 3),
           "call_ms": [round(1e3 * x, 2) for x in per_step],
           "device_ms": [round(1e3 * x[1], 2) for x in parts],
           "h2d_bytes_per_step": int(n_e * plan.nnz * 16 + plan.nnz * 16),
           "d2h_bytes_per_step": int(2 * n_e * plan.n * 16),
           "api": "paper_1104_0623_b200.solve_batch(mesh, [SparseOperator]*16, Sigma, SolverConfig())"}

    flops_total = 8.0 * W * n_e * world * args.steps / (dev_ms * 1e-3) / 1e12
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": f"cfg{args.config}: {cfg.nx}x{cfg.ny} {cfg.stencil}-point stencil + dense contacts, "
                               f"{n_e} energy points per GPU, diag G^r + G^<",
                   "mesh": [cfg.nx, cfg.ny], "n_energies_per_gpu": n_e, "stencil": cfg.stencil,
                   "parallelism": f"replicas{world} (energy sharding)" if world > 1 else "single GPU",
                   "l2": "flushed (256 MiB write) between timed steps, outside the timed events",
                   "launch": ("CUDA graph replay of the solve's launch schedule" if graph is not None
                              else "direct launches")},
        "fp64_tflops": flops_total, "fp64_frac_of_peak": flops_total / FP64_PEAK_TFLOPS,
        "work_per_energy_mults": W,
        "roofline": roofline,
        "near_root": near_root,
        "kernels": kernels,
        "e2e": e2e,
        "gpu_launches": int(plan.launch_count(n_e) * args.steps),
        "clocks": clk,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_line(args.config, config_problem(args.config, 1))
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
