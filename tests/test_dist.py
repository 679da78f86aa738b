"""World-size-2 gloo test of the energy-sharded (replica) path, CPU only: the
per-rank solver is the CPU oracle, so this exercises sharding and the gather."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, outdir):
    import sys

    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist

    from oracle.find_oracle import FindOracle
    from paper_1104_0623_b200 import Mesh, SolverConfig, SparseOperator
    from paper_1104_0623_b200.configs import build_problem
    from paper_1104_0623_b200.dist import solve_batch_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = build_problem(6, 5, np.linspace(0.5, 3.5, 5), seed=4)
    mesh = Mesh(p.nx, p.ny)
    ops = [SparseOperator(p.a_csr(k)) for k in range(p.energies.size)]

    class R:
        pass

    def oracle_solver(mesh, a_sub, sigma, config):
        o = FindOracle(mesh.nx, mesh.ny, a_sub[0].matrix)
        rs = [o.solve(a.matrix, sigma.matrix) for a in a_sub]
        r = R()
        r.gr_diag = np.array([x.gr_diag for x in rs]).reshape(len(a_sub), -1)
        r.gless_diag = np.array([x.gless_diag for x in rs]).reshape(len(a_sub), -1)
        return r

    gr, gl = solve_batch_sharded(mesh, ops, SparseOperator(p.sigma_csr()), SolverConfig(), local_solver=oracle_solver)
    np.save(os.path.join(outdir, f"gr{rank}.npy"), gr)
    np.save(os.path.join(outdir, f"gl{rank}.npy"), gl)
    dist.destroy_process_group()


def test_energy_shard_balanced():
    from paper_1104_0623_b200.dist import energy_shard

    for n in range(0, 13):
        for w in range(1, 5):
            sl = [energy_shard(n, r, w) for r in range(w)]
            assert sl[0].start == 0 and sl[-1].stop == n
            assert all(a.stop == b.start for a, b in zip(sl, sl[1:]))
            assert max(s.stop - s.start for s in sl) - min(s.stop - s.start for s in sl) <= 1
    with pytest.raises(ValueError):
        energy_shard(4, 2, 2)


def test_sharded_solve_gloo_world2(tmp_path):
    from oracle.find_oracle import FindOracle
    from paper_1104_0623_b200.configs import build_problem

    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    p = build_problem(6, 5, np.linspace(0.5, 3.5, 5), seed=4)
    o = FindOracle(p.nx, p.ny, p.a_csr(0))
    ref = [o.solve(p.a_csr(k), p.sigma_csr()) for k in range(p.energies.size)]
    for rank in range(2):
        gr = np.load(tmp_path / f"gr{rank}.npy")
        gl = np.load(tmp_path / f"gl{rank}.npy")
        assert gr.shape == (5, p.n)
        for k in range(5):
            np.testing.assert_array_equal(gr[k], ref[k].gr_diag)
            np.testing.assert_array_equal(gl[k], ref[k].gless_diag)


def test_balanced_chunk_arithmetic():
    """Energy points per find_solve call: capped by the fit and by grid.y's 0xffff, balanced."""
    from paper_1104_0623_b200.solver import MAX_ENERGIES_PER_LAUNCH, balanced_chunk

    assert balanced_chunk(8, 7) == 4 and balanced_chunk(8, 8) == 8 and balanced_chunk(8, 100) == 8
    assert balanced_chunk(5, 0) == 1 and balanced_chunk(1, 1) == 1
    big = 3 * MAX_ENERGIES_PER_LAUNCH + 5
    c = balanced_chunk(big, 10 ** 9)
    assert c <= MAX_ENERGIES_PER_LAUNCH and -(-big // c) == 4  # four balanced calls, none above the limit
    for n in range(1, 40):
        for fit in range(1, 12):
            c = balanced_chunk(n, fit)
            calls = -(-n // c)
            assert c <= fit and calls == -(-n // min(fit, n))


def _worker_small(rank, world, port, outdir):
    import sys

    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist

    from oracle.find_oracle import FindOracle
    from paper_1104_0623_b200 import Mesh, SolverConfig, SparseOperator
    from paper_1104_0623_b200.configs import build_problem
    from paper_1104_0623_b200.dist import solve_batch_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = build_problem(5, 4, [1.1], seed=6)
    mesh = Mesh(p.nx, p.ny)
    calls = []

    class R:
        pass

    def oracle_solver(mesh, a_sub, sigma, config):
        calls.append(len(a_sub))
        o = FindOracle(mesh.nx, mesh.ny, a_sub[0].matrix)
        rs = [o.solve(a.matrix, sigma.matrix) for a in a_sub]
        r = R()
        r.gr_diag = np.array([x.gr_diag for x in rs]).reshape(len(a_sub), -1)
        r.gless_diag = np.array([x.gless_diag for x in rs]).reshape(len(a_sub), -1)
        return r

    gr, gl = solve_batch_sharded(mesh, [SparseOperator(p.a_csr(0))], SparseOperator(p.sigma_csr()), SolverConfig(),
                                 local_solver=oracle_solver)
    np.save(os.path.join(outdir, f"gr{rank}.npy"), gr)
    np.save(os.path.join(outdir, f"calls{rank}.npy"), np.array(calls))
    dist.destroy_process_group()


def test_sharded_solve_more_ranks_than_energies(tmp_path):
    """World 2, one energy point: rank 1 has an empty shard, joins the gathers without solving."""
    from oracle.find_oracle import FindOracle
    from paper_1104_0623_b200.configs import build_problem

    mp.spawn(_worker_small, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    p = build_problem(5, 4, [1.1], seed=6)
    ref = FindOracle(p.nx, p.ny, p.a_csr(0)).solve(p.a_csr(0), p.sigma_csr())
    for rank in range(2):
        np.testing.assert_array_equal(np.load(tmp_path / f"gr{rank}.npy")[0], ref.gr_diag)
    assert list(np.load(tmp_path / "calls0.npy")) == [1] and list(np.load(tmp_path / "calls1.npy")) == []


@pytest.mark.gpu
def test_sharded_solve_gpu_world1(cuda):
    """solve_batch_sharded with the real GPU solve_batch (world size 1, gloo), against the oracle."""
    import torch.distributed as dist

    from oracle.find_oracle import FindOracle
    from paper_1104_0623_b200 import Mesh, SolverConfig, SparseOperator
    from paper_1104_0623_b200.configs import build_problem
    from paper_1104_0623_b200.dist import solve_batch_sharded

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        p = build_problem(9, 7, np.linspace(0.5, 3.5, 3), seed=8)
        ops = [SparseOperator(p.a_csr(k)) for k in range(3)]
        gr, gl = solve_batch_sharded(Mesh(p.nx, p.ny), ops, SparseOperator(p.sigma_csr()), SolverConfig())
    finally:
        dist.destroy_process_group()
    o = FindOracle(p.nx, p.ny, p.a_csr(0))
    for k in range(3):
        r = o.solve(p.a_csr(k), p.sigma_csr())
        assert np.abs(gr[k] - r.gr_diag).max() <= 1e-10 * np.abs(r.gr_diag).max()
        assert np.abs(gl[k] - r.gless_diag).max() <= 1e-10 * np.abs(r.gless_diag).max()
