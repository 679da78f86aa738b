"""Drop-in ``solve`` on the B200 path (mirror of find_selinv/solver.py:53-89, 586-701).

Same signature, validation, error types and result fields as the reference;
the arithmetic runs in the sm_100a kernels behind the C ABI (include/find_b200.h).
There is no CPU fallback: without a CUDA device the call raises.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp

from .errors import NativeLibraryError, StructureMismatchError
from .ledger import BLOCK_KERNELS, HERMITIAN_KERNELS, KERNEL_NAMES, FlopLedger
from .operators import check_pattern_subset, check_structural_symmetry, is_hermitian
from .plan import Plan, plan_for, same_array


@dataclass
class SolverConfig:
    """solver.py:53-71 (same fields, defaults and validation)."""

    kernel: str = "naive"
    use_symmetry: bool = False
    compute_gless: bool = True
    compute_offdiag: bool = False
    tiling: str = "full-leaves"
    leaf_max: int = 2
    pivot_rtol: float = 1e-12
    sigma_mode: str = "auto"
    debug_checks: bool = False

    def __post_init__(self):
        if self.kernel not in KERNEL_NAMES:
            raise ValueError(f"unknown kernel {self.kernel!r}; choose from {KERNEL_NAMES}")
        if self.tiling not in ("full-leaves", "half-leaves"):
            raise ValueError(f"unknown tiling {self.tiling!r}")
        if self.kernel in HERMITIAN_KERNELS:
            self.use_symmetry = True


@dataclass
class SelectedInverse:
    """solver.py:82-89."""

    gr_diag: np.ndarray
    gless_diag: np.ndarray | None
    offdiag: dict | None
    ledger: FlopLedger
    timings: dict = field(default_factory=dict)
    stats: dict = field(default_factory=dict)
    # beyond the reference fields: G^< on the same adjacent pairs as ``offdiag`` (the
    # reference computes these only inside _extended_extraction, solver.py:487-507)
    offdiag_gless: dict | None = None


@dataclass
class SelectedInverseBatch:
    """Result of :func:`solve_batch`: one row per energy point."""

    gr_diag: np.ndarray  # [nE, n]
    gless_diag: np.ndarray | None
    ledger: FlopLedger  # per energy point
    timings: dict = field(default_factory=dict)
    stats: dict = field(default_factory=dict)
    offdiag_pairs: np.ndarray | None = None  # [n_pairs, 2] directed adjacent pairs (u, v), ascending
    offdiag_gr: np.ndarray | None = None     # [nE, n_pairs] G^r(u, v)
    offdiag_gless: np.ndarray | None = None  # [nE, n_pairs] G^<(u, v)


def _csr_sorted(m) -> sp.csr_matrix:
    m = m.tocsr()
    if not m.has_sorted_indices:
        m = m.copy()
        m.sort_indices()
    return m


def sigma_on_pattern(a: sp.csr_matrix, sigma: sp.csr_matrix) -> np.ndarray:
    """Sigma values scattered onto A's CSR slots (zeros where Sigma has no entry)."""
    n = a.shape[0]
    rows_a = np.repeat(np.arange(n, dtype=np.int64), np.diff(a.indptr))
    keys = rows_a * n + a.indices.astype(np.int64)
    s = sigma.tocoo()
    skeys = s.row.astype(np.int64) * n + s.col.astype(np.int64)
    pos = np.searchsorted(keys, skeys)
    ok = (pos < keys.size) & (keys[np.minimum(pos, keys.size - 1)] == skeys)
    if not ok.all():
        raise ValueError("scattering pattern exceeds the operator pattern")
    out = np.zeros(a.nnz, np.complex128)
    np.add.at(out, pos, s.data.astype(np.complex128))
    return out


def sigma_symmetry(sigma_csr) -> int:
    """+1 if exactly Hermitian, -1 if exactly skew-Hermitian, else 0."""
    m = sigma_csr.tocsr()
    h = m.conj().T.tocsr()
    if (m - h).count_nonzero() == 0:
        return 1
    if (m + h).count_nonzero() == 0:
        return -1
    return 0


def _transpose_slots(plan: Plan) -> np.ndarray:
    """CSR slot of (j, i) for every slot (i, j) of the (structurally symmetric) pattern; cached per plan."""
    t = plan.cache.get("tslots")
    if t is None:
        n = plan.n
        rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(plan.indptr))
        keys = rows * n + plan.indices
        t = np.searchsorted(keys, plan.indices * n + rows)
        plan.cache["tslots"] = t
    return t


def _sigma_prepare(plan: Plan, am: sp.csr_matrix, sigma) -> tuple[np.ndarray, int, bool]:
    """Sigma on A's pattern, its exact (skew-)Hermitian symmetry, and the reference's
    tolerance-based is_hermitian (operators.py:98-103).  The result of the last call is
    reused when Sigma's pattern and values are bit-identical (three memcmp-speed
    comparisons), as in an energy sweep that passes the same Sigma every time."""
    sm = _csr_sorted(sigma.matrix)
    last = plan.cache.get("sigma_last")
    if (last is not None and last[0].size == sm.indptr.size and last[1].size == sm.indices.size
            and same_array(last[0], sm.indptr) and same_array(last[1], sm.indices)
            and np.array_equal(last[2], sm.data)):
        return last[3]
    out = _sigma_prepare_full(plan, sm)
    plan.cache["sigma_last"] = (sm.indptr.copy(), sm.indices.copy(), sm.data.copy(), out)
    return out


def _sigma_prepare_full(plan: Plan, sm: sp.csr_matrix) -> tuple[np.ndarray, int, bool]:
    import hashlib

    h = hashlib.sha1(np.ascontiguousarray(sm.indptr, np.int64).tobytes())
    h.update(np.ascontiguousarray(sm.indices, np.int64).tobytes())
    key = ("sigma_slots", h.hexdigest())
    slots = plan.cache.get(key)
    if slots is None:
        n = plan.n
        rows_a = np.repeat(np.arange(n, dtype=np.int64), np.diff(plan.indptr))
        keys = rows_a * n + plan.indices
        srows = np.repeat(np.arange(n, dtype=np.int64), np.diff(sm.indptr))
        skeys = srows * n + sm.indices.astype(np.int64)
        slots = np.searchsorted(keys, skeys)
        ok = (slots < keys.size) & (keys[np.minimum(slots, keys.size - 1)] == skeys)
        if not ok.all():
            raise ValueError("scattering pattern exceeds the operator pattern")
        plan.cache[key] = slots
    s_vals = np.zeros(plan.nnz, np.complex128)
    s_vals[slots] = sm.data
    t = _transpose_slots(plan)
    st = np.conj(s_vals[t])
    sym = 1 if np.array_equal(s_vals, st) else (-1 if np.array_equal(s_vals, -st) else 0)
    scale = np.abs(sm.data).max() if sm.nnz else 1.0
    herm = bool(np.abs(s_vals - st).max() <= 1e-12 * max(scale, 1.0)) if s_vals.size else True
    return s_vals, sym, herm


def _validate(mesh, a, sigma, config, plan_cache: dict | None = None):
    """solver.py:591-608 (pattern-only checks are cached per plan)."""
    if a.n != mesh.n:
        raise ValueError(f"operator size {a.n} does not match mesh with {mesh.n} nodes")
    if plan_cache is None or not plan_cache.get("structurally_symmetric"):
        if not check_structural_symmetry(a):
            raise ValueError("operator pattern is not structurally symmetric")
        if plan_cache is not None:
            plan_cache["structurally_symmetric"] = True
    if config.compute_gless:
        if sigma is None:
            raise ValueError("compute_gless requires a scattering matrix")
        if sigma.n != a.n:
            raise ValueError("scattering matrix size mismatch")
        if plan_cache is None and not check_pattern_subset(sigma, a):
            raise ValueError("scattering pattern exceeds the operator pattern")
    if config.kernel == "ldlt":
        d = a.matrix - a.matrix.T
        scale = max(np.abs(a.matrix.data).max() if a.matrix.nnz else 1.0, 1.0)
        if d.nnz and np.abs(d.data).max() > 1e-10 * scale:
            raise ValueError("ldlt kernel requires a (complex-)symmetric operator")
    elif config.use_symmetry and not is_hermitian(a.matrix):
        raise ValueError("use_symmetry requires a Hermitian operator")


def _device():
    import torch

    if not torch.cuda.is_available():
        raise NativeLibraryError("the FIND B200 path needs a CUDA device (there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


MAX_ENERGIES_PER_LAUNCH = 0xFFFF  # grid.y carries the energy index (find_solve rejects more)


def balanced_chunk(n_e: int, fit: int) -> int:
    """Energy points per find_solve call: at most ``fit`` (what the device memory holds) and
    MAX_ENERGIES_PER_LAUNCH, balanced over the calls (8 points at <= 7 per call -> 4 + 4)."""
    chunk = max(1, min(n_e, int(fit), MAX_ENERGIES_PER_LAUNCH))
    return -(-n_e // -(-n_e // chunk))


def energy_chunk(plan: Plan, n_e: int, compute_gless: bool, dev, n_pairs: int = 0) -> int:
    """Energy points per find_solve call that fit in 90 % of the free device memory (the plan's
    own cached workspace counts as free), inputs / outputs included."""
    import torch

    per_energy = plan.workspace_bytes(2, compute_gless) - plan.workspace_bytes(1, compute_gless)
    per_energy += (plan.nnz + 2 * plan.n) * 16 + 2 * n_pairs * 16
    free, total = torch.cuda.mem_get_info(dev)
    held = plan._ws.numel() if plan._ws is not None and plan._ws.device == dev else 0
    if free + held < 0.5 * total:  # other plans' cached workspaces crowd this solve out
        from .plan import release_workspaces

        release_workspaces(keep=plan)
        free, total = torch.cuda.mem_get_info(dev)
    fit = (0.90 * (free + held) - plan.workspace_bytes(1, compute_gless) + per_energy) // per_energy
    return balanced_chunk(n_e, fit)


def solve_values(plan: Plan, a_vals: np.ndarray, s_vals: np.ndarray | None, compute_gless=True, pivot_rtol=1e-12,
                 sigma_sym=0, max_chunk: int | None = None, compute_offdiag=False, offdiag_out: dict | None = None,
                 host_work=None):
    """Run the plan on host value arrays a_vals [nE, nnz], s_vals [nnz] or [nE, nnz].

    Energy points are processed in chunks sized to the free device memory (one
    find_solve per chunk); per chunk: host -> device copies, the level-batched
    kernels, status check, device -> host copy of the diagonals.
    With compute_offdiag, G^r (and G^< when compute_gless) on plan.offdiag_pairs() are
    stored into offdiag_out["gr"] / ["gl"] ([nE, n_pairs]).
    host_work: optional callable run once while the first chunk executes on the device.
    Returns (gr, gl, device_seconds_up, device_seconds_down)."""
    import torch

    dev = _device()
    a_vals = np.ascontiguousarray(np.atleast_2d(a_vals), dtype=np.complex128)
    n_e = a_vals.shape[0]
    s_b = True
    if compute_gless:
        s_vals = np.ascontiguousarray(s_vals, dtype=np.complex128)
        s_b = s_vals.ndim == 1
    n_pairs = plan.offdiag_pairs().shape[0] if compute_offdiag else 0
    chunk = energy_chunk(plan, n_e, compute_gless, dev, n_pairs)
    if max_chunk:
        chunk = balanced_chunk(n_e, min(chunk, max_chunk))
    # the plan's own (non-default) stream, ordered after the caller's current stream; every chunk
    # ends with a host synchronisation, so the caller's stream needs no wait afterwards
    stream = plan.solve_stream(dev)
    stream.wait_stream(torch.cuda.current_stream(dev))
    gr = np.empty((n_e, plan.n), np.complex128)
    gl = np.empty((n_e, plan.n), np.complex128) if compute_gless else None
    s_all = torch.from_numpy(s_vals) if (compute_gless and s_b) else None
    a_host = plan.pinned_tensor(a_vals) if plan.is_pinned_view(a_vals) else torch.from_numpy(a_vals)
    if compute_offdiag:
        offdiag_out["gr"] = np.empty((n_e, n_pairs), np.complex128)
        offdiag_out["gl"] = np.empty((n_e, n_pairs), np.complex128) if compute_gless else None
    t_up = t_down = 0.0
    with torch.cuda.stream(stream):  # copies, events and kernels all on the plan's stream
        for k0 in range(0, n_e, chunk):
            k1 = min(n_e, k0 + chunk)
            c = k1 - k0
            # inputs / outputs in plan-owned device buffers: fixed addresses, so the level schedule
            # is captured once as a CUDA graph and replayed (Plan.replay_or_run)
            a_d = plan.device_buffer("a", (c, plan.nnz), dev)
            a_d.copy_(a_host[k0:k1], non_blocking=True)
            s_d = None
            if compute_gless:
                s_d = plan.device_buffer("s", (plan.nnz,) if s_b else (c, plan.nnz), dev)
                s_d.copy_(s_all if s_b else torch.from_numpy(s_vals[k0:k1]), non_blocking=True)
            gr_d = plan.device_buffer("gr", (c, plan.n), dev)
            gl_d = plan.device_buffer("gl", (c, plan.n), dev) if compute_gless else None
            og_d = ol_d = None
            if compute_offdiag:
                og_d = plan.device_buffer("og", (c, max(n_pairs, 1)), dev)
                ol_d = plan.device_buffer("ol", (c, max(n_pairs, 1)), dev) if compute_gless else None
            ws = plan.workspace(c, compute_gless, dev)
            key = (c, int(compute_gless), int(s_b), int(sigma_sym), float(pivot_rtol), bool(compute_offdiag),
                   ws.data_ptr(), stream.cuda_stream)
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
            ev[0].record(stream)
            plan.replay_or_run(("up",) + key, stream, lambda: plan.run(
                a_d, s_d, gr_d, gl_d, compute_gless, pivot_rtol, s_b, ws=ws, stream=stream,
                groups=(0, plan.first_down_group), sigma_sym=sigma_sym))
            ev[1].record(stream)
            plan.replay_or_run(("down",) + key, stream, lambda: plan.run(
                a_d, s_d, gr_d, gl_d, compute_gless, pivot_rtol, s_b, ws=ws, stream=stream,
                groups=(plan.first_down_group, -1), sigma_sym=sigma_sym, off_gr=og_d, off_gl=ol_d))
            ev[2].record(stream)
            out_h = plan.host_outputs(k1 - k0, compute_gless)
            out_h[0].copy_(gr_d, non_blocking=True)
            if compute_gless:
                out_h[1].copy_(gl_d, non_blocking=True)
            if host_work is not None and k0 == 0:
                host_work()
            try:
                plan.check_status(ws, k1 - k0, stream)
            except Exception as exc:
                if hasattr(exc, "energy") and exc.energy is not None:
                    exc.energy += k0
                raise
            gr[k0:k1] = out_h[0].numpy()
            if compute_gless:
                gl[k0:k1] = out_h[1].numpy()
            if compute_offdiag:
                offdiag_out["gr"][k0:k1] = og_d[:, :n_pairs].cpu().numpy()
                if compute_gless:
                    offdiag_out["gl"][k0:k1] = ol_d[:, :n_pairs].cpu().numpy()
            t_up += ev[0].elapsed_time(ev[1]) * 1e-3
            t_down += ev[1].elapsed_time(ev[2]) * 1e-3
    return gr, gl, t_up, t_down


def _stats(plan: Plan, a_data: np.ndarray) -> dict:
    """solver.py:186, 217-219: structure-exception entries of A that are nonzero."""
    occ = plan.cache.get("exception_occ")
    if occ is None:  # how often each CSR slot is an exception entry, per pass
        occ = tuple(np.bincount(plan.exception_slots(k), minlength=plan.nnz).astype(np.int64) for k in (0, 1))
        plan.cache["exception_occ"] = occ
    f = a_data.view(np.float64)
    nz = (f[0::2] != 0) | (f[1::2] != 0)
    return {
        "upward_exception_entries": int(np.dot(nz, occ[0])),
        "downward_exception_entries": int(np.dot(nz, occ[1])),
    }


def _leaf_table(plan: Plan):
    """(final-step indices, leaf rectangles [x0, y0, w, h]) in plan order, cached."""
    t = plan.cache.get("leaf_table")
    if t is None:
        fin = np.nonzero(plan.kind == 3)[0]
        rect = np.zeros((fin.size, 4), np.int64)
        for i, k in enumerate(fin):
            nodes = plan.cluster_set(int(plan.label[k]), 0)
            x, y = nodes % plan.nx, nodes // plan.nx
            rect[i] = (x.min(), y.min(), x.max() - x.min() + 1, y.max() - y.min() + 1)
        t = (fin, rect)
        plan.cache["leaf_table"] = t
    return t


def half_leaves_selection(plan: Plan):
    """select_tiling(tree, "half-leaves") (solver.py:522-556): boolean mask over the final
    steps, or None when the reference falls back to full-leaves (with its warning)."""
    import warnings

    fin, rect = _leaf_table(plan)
    shapes = {(int(w), int(h)) for w, h in rect[:, 2:]}
    if len(shapes) != 1:
        warnings.warn("non-uniform leaves; falling back to full-leaves tiling")
        return None
    lw, lh = shapes.pop()
    if max(lw, lh) > 2:
        warnings.warn("half-leaves tiling needs leaves of side <= 2; using full-leaves")
        return None
    ntx, nty = plan.nx // lw, plan.ny // lh
    ti, tj = rect[:, 0] // lw, rect[:, 1] // lh
    on_edge = (ti == 0) | (tj == 0) | (ti == ntx - 1) | (tj == nty - 1)
    return on_edge | ((ti + tj) % 2 == 0)


def _ledger_cached(plan: Plan, config, sigma_herm: bool) -> FlopLedger:
    """The reference's FlopLedger for this config: merges as charged by the kernel
    dispatch; leaf extraction as full-leaves (final step, inverse, sandwich and, with
    compute_offdiag, offdiag_backsub, solver.py:475) or half-leaves (one dense inverse
    and sandwich of ring+leaf per selected leaf, solver.py:487-507)."""
    half = config.tiling == "half-leaves"
    key = ("ledger", config.kernel, bool(config.compute_gless), bool(sigma_herm), config.sigma_mode,
           bool(config.compute_offdiag), half)
    led = plan.cache.get(key)
    if led is None:
        sel = half_leaves_selection(plan) if half else None
        if sel is None:
            led = plan.ledger(config.kernel, config.compute_gless, sigma_herm, config.sigma_mode)
            if config.compute_offdiag:
                fin = plan.kind == 3
                t = plan.s[fin].astype(object)
                c = plan.b[fin].astype(object)
                m = t > 0
                if m.any():
                    led.add("offdiag_backsub", 2 * int(np.sum(t[m] ** 2 * c[m] + t[m] * c[m] ** 2)))
        else:
            from .ledger import plan_ledger

            nf = plan.kind != 3
            led = plan_ledger(plan.kind[nf], plan.s[nf], plan.b[nf], config.kernel, config.compute_gless, sigma_herm,
                              config.sigma_mode)
            fin, _ = _leaf_table(plan)
            m = (plan.s[fin] + plan.b[fin])[sel].astype(object)
            led.add("dense_inverse", int(np.sum(m ** 3)))
            if config.compute_gless:
                led.add("gless_sandwich", 2 * int(np.sum(m ** 3)))
        plan.cache[key] = led
    return FlopLedger(led.multiplications, dict(led.by_kernel))


def _offdiag_dict(pairs: np.ndarray, vals: np.ndarray) -> dict:
    return dict(zip(map(tuple, pairs.tolist()), vals.tolist()))


def _prepare(mesh, a_list, sigma, config):
    """Validation (solver.py:591-608), cached plan, values packed into a reused pinned buffer."""
    if not a_list:
        raise ValueError("a_list is empty")
    if a_list[0].n != mesh.n:
        raise ValueError(f"operator size {a_list[0].n} does not match mesh with {mesh.n} nodes")
    am0 = _csr_sorted(a_list[0].matrix)
    plan, _ = plan_for(mesh.nx, mesh.ny, am0.indptr, am0.indices, config.leaf_max)
    _validate(mesh, a_list[0], sigma, config, plan.cache)
    import torch

    vals = plan.host_values(len(a_list))
    vt = plan.pinned_tensor(vals)  # the same pinned buffer as a tensor: torch's multi-threaded copies
    for k, a in enumerate(a_list):
        am = am0 if k == 0 else _csr_sorted(a.matrix)
        if am.nnz != am0.nnz or not same_array(am.indptr, am0.indptr) or not same_array(am.indices, am0.indices):
            raise ValueError("all operators of a batch must share one sparsity pattern")
        vt[k].copy_(torch.from_numpy(np.ascontiguousarray(am.data)))
    s_vals, ssym, sherm = (None, 0, False)
    if config.compute_gless:
        s_vals, ssym, sherm = _sigma_prepare(plan, am0, sigma)
    elif sigma is not None:
        sherm = is_hermitian(sigma.matrix)
    return plan, am0, vals, s_vals, ssym, sherm


def _debug_checks(config, stats: dict) -> None:
    """debug_checks (solver.py:136, 156): the structured kernels refuse upward merges whose
    inputs violate the merge sparsity structure (kernels.py:350-355 _check_strict)."""
    if not config.debug_checks:
        return
    if config.kernel in BLOCK_KERNELS or config.kernel == "symmetric_sparse":
        bad = int(stats.get("upward_exception_entries", 0))
        if bad:
            raise StructureMismatchError(f"{bad} entries violate the merge sparsity structure")


def solve(mesh, a, sigma, config: SolverConfig) -> SelectedInverse:
    """Run the full selected inversion on one operator (solver.py:586-701)."""
    t0 = time.perf_counter()
    plan, am, vals, s_vals, ssym, sherm = _prepare(mesh, [a], sigma, config)
    t1 = time.perf_counter()
    off = {}
    side = {}
    gr, gl, t_up, t_down = solve_values(plan, vals, s_vals, config.compute_gless, config.pivot_rtol, ssym,
                                        compute_offdiag=config.compute_offdiag, offdiag_out=off,
                                        host_work=lambda: side.update(stats=_stats(plan, am.data)))
    _debug_checks(config, side["stats"])
    led = _ledger_cached(plan, config, sherm)
    offd = offl = None
    if config.compute_offdiag:
        pairs = plan.offdiag_pairs()
        offd = _offdiag_dict(pairs, off["gr"][0])
        if off.get("gl") is not None:
            offl = _offdiag_dict(pairs, off["gl"][0])
    t3 = time.perf_counter()
    return SelectedInverse(
        gr_diag=gr[0],
        gless_diag=gl[0] if gl is not None else None,
        offdiag=offd,
        ledger=led,
        timings={"tree": t1 - t0, "upward": t_up, "downward_extract": t_down, "total": t3 - t0},
        stats=side["stats"],
        offdiag_gless=offl,
    )


def solve_batch(mesh, a_list, sigma, config: SolverConfig) -> SelectedInverseBatch:
    """Energy-batched solve: every operator shares A's pattern; one launch per
    (tree level, size class) covers all energy points."""
    t0 = time.perf_counter()
    plan, am0, vals, s_vals, ssym, sherm = _prepare(mesh, list(a_list), sigma, config)
    t1 = time.perf_counter()
    off = {}
    side = {}
    gr, gl, t_up, t_down = solve_values(plan, vals, s_vals, config.compute_gless, config.pivot_rtol, ssym,
                                        compute_offdiag=config.compute_offdiag, offdiag_out=off,
                                        host_work=lambda: side.update(stats=_stats(plan, am0.data),
                                                                      ledger=_ledger_cached(plan, config, sherm)))
    _debug_checks(config, side["stats"])
    t3 = time.perf_counter()
    res = SelectedInverseBatch(gr, gl, side["ledger"],
                               {"tree": t1 - t0, "upward": t_up, "downward_extract": t_down, "total": t3 - t0},
                               side["stats"])
    if config.compute_offdiag:
        res.offdiag_pairs = plan.offdiag_pairs()
        res.offdiag_gr = off["gr"]
        res.offdiag_gless = off.get("gl")
    return res
