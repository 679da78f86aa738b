"""Multi-GPU energy sharding (replicas only).

Energy points are independent and share one plan, so N processes (one per GPU,
torch.distributed) each solve a contiguous shard of the energy list; the only
exchange is an all-gather of the 2*n diagonal entries per energy point.
"""

from __future__ import annotations

import numpy as np


def energy_shard(n_energies: int, rank: int, world: int) -> slice:
    """Contiguous, balanced shard of range(n_energies) for `rank` (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("invalid rank / world size")
    base, extra = divmod(n_energies, world)
    start = rank * base + min(rank, extra)
    return slice(start, start + base + (1 if rank < extra else 0))


def _gather_rows(local: np.ndarray, n_total: int, n_cols: int, group=None) -> np.ndarray:
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    sizes = [energy_shard(n_total, r, world) for r in range(world)]
    width = max(s.stop - s.start for s in sizes)
    buf = np.zeros((width, n_cols, 2), np.float64)
    buf[: local.shape[0]] = local.view(np.float64).reshape(local.shape[0], n_cols, 2)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.from_numpy(buf).to(dev)
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t, group=group)
    full = np.empty((n_total, n_cols), np.complex128)
    for r, s in enumerate(sizes):
        part = outs[r].cpu().numpy()[: s.stop - s.start]
        full[s] = part[..., 0] + 1j * part[..., 1]
    return full


def solve_batch_sharded(mesh, a_list, sigma, config, group=None, local_solver=None):
    """Each rank solves its energy shard; diagonals are all-gathered to every rank.

    `local_solver(mesh, a_sublist, sigma, config)` must return an object with
    `gr_diag` [k, n] and `gless_diag` [k, n] (default: `solve_batch`)."""
    import torch.distributed as dist

    if local_solver is None:
        from .solver import solve_batch as local_solver
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if not a_list:
        raise ValueError("a_list is empty")  # every rank sees the same list: all raise, none blocks
    sl = energy_shard(len(a_list), rank, world)
    n = mesh.n
    if sl.stop > sl.start:
        res = local_solver(mesh, a_list[sl], sigma, config)
        gr_l = np.asarray(res.gr_diag).reshape(-1, n)
        gl_l = np.asarray(res.gless_diag).reshape(-1, n) if config.compute_gless else None
    else:  # more ranks than energy points: this rank only joins the gathers
        gr_l = np.zeros((0, n), np.complex128)
        gl_l = np.zeros((0, n), np.complex128)
    gr = _gather_rows(gr_l, len(a_list), n, group)
    gl = _gather_rows(gl_l, len(a_list), n, group) if config.compute_gless else None
    return gr, gl
