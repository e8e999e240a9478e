"""Direction-sharded lattice operator (moment layout, configs 4-5): host logic on CPU ranks
(gloo, world_size 2) with the oracle standing in for the device halves, and the direction
partition.  The device halves (rtk_lattice_partial_moments / rtk_lattice_apply_with_moments)
are checked on the GPU in tests/test_gpu_sharding.py."""
import os
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


class OracleLatticeShardOps:
    """Oracle restatement of the two device halves (test infrastructure only)."""

    def __init__(self, problem, a0, a1):
        from oracle import lattice as OL

        self.OL = OL
        self.d = OL.desc_from_lattice_problem(problem)
        self.a0, self.a1 = a0, a1

    def partial_moments(self, u):
        import torch

        d, OL = self.d, self.OL
        I = OL.lattice_transfer(d, OL.source_from_moments(d, np.asarray(u, dtype=float)))
        w = (d.ybasis * d.dir_w[None, :])[:, self.a0:self.a1]
        m = np.einsum("ka,saf->skf", w, I.reshape(d.n_space, d.n_dirs, d.n_freq)[:, self.a0:self.a1, :])
        return torch.from_numpy(m.reshape(-1).copy())

    def apply_with_moments(self, u, m):
        import torch

        d = self.d
        Rm = self.OL.redistribute(d, np.asarray(m, dtype=float).reshape(d.n_space, d.n_mom, d.n_freq))
        return torch.from_numpy(np.asarray(u, dtype=float) - Rm.reshape(-1))


def _problem():
    sys.path.insert(0, ROOT)
    from paper_2602_21958_b200 import lattice as L

    return L.lattice_problem(5, 4, 6, 8, 6, 3, corr_len=2.0, seed=4, layout="moments", characteristics="hybrid")


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from oracle import lattice as OL
    from oracle import rt_oracle as ro
    from paper_2602_21958_b200.sharding import LatticeShardedOperator

    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = _problem()
    op = LatticeShardedOperator(p, ops_factory=OracleLatticeShardOps)
    u = torch.from_numpy(np.random.default_rng(3).standard_normal(p.n_total))
    y = op(u)
    d = OL.desc_from_lattice_problem(p)
    b = OL.build_rhs(d, "moments")
    rep = ro.gmres(lambda v: op(torch.from_numpy(np.asarray(v, dtype=float))).numpy(), b, rel_tol=1e-9, max_iter=300)
    q.put((rank, (op.a0, op.a1), y.numpy().tolist(), rep.iterations, rep.solution.tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(240)
def test_two_ranks_reproduce_the_lattice_operator_and_gmres():
    """The all-reduced partial moments give apply_A on every rank, and a solver run
    redundantly on the replicated vectors takes the single-process path."""
    from oracle import lattice as OL
    from oracle import rt_oracle as ro

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29800 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    out = sorted(q.get(timeout=200) for _ in procs)
    for pr in procs:
        pr.join(timeout=30)
    assert all(pr.exitcode == 0 for pr in procs)
    p = _problem()
    d = OL.desc_from_lattice_problem(p)
    u = np.random.default_rng(3).standard_normal(p.n_total)
    ref = OL.apply_A_moments(d, u)
    assert out[0][1][0] == 0 and out[0][1][1] == out[1][1][0] and out[1][1][1] == p.n_dirs
    for _, _, y, _, _ in out:
        assert np.linalg.norm(np.asarray(y) - ref) <= 1e-13 * np.linalg.norm(ref)
    np.testing.assert_array_equal(np.asarray(out[0][2]), np.asarray(out[1][2]))   # same bits on every rank
    b = OL.build_rhs(d, "moments")
    single = ro.gmres(lambda v: OL.apply_A_moments(d, v), b, rel_tol=1e-9, max_iter=300)
    assert out[0][3] == out[1][3] and abs(out[0][3] - single.iterations) <= 1
    sol = np.asarray(single.solution)
    assert np.linalg.norm(np.asarray(out[0][4]) - sol) <= 1e-7 * np.linalg.norm(sol)


def test_direction_blocks_balance_the_transfer_cost():
    sys.path.insert(0, ROOT)
    from paper_2602_21958_b200 import lattice as L
    from paper_2602_21958_b200.sharding import direction_blocks, lattice_direction_cost

    p = L.lattice_problem(8, 8, 6, 8, 12, 4, layout="moments")
    cost = lattice_direction_cost(p)
    assert cost.size == p.n_dirs and cost.min() >= 2
    for world in (1, 2, 3, 4, 8):
        blocks = direction_blocks(cost, world)
        assert blocks[0][0] == 0 and blocks[-1][1] == p.n_dirs
        assert all(b0 < b1 for b0, b1 in blocks) and all(blocks[r][1] == blocks[r + 1][0] for r in range(world - 1))
        loads = [cost[a:b].sum() for a, b in blocks]
        assert max(loads) <= cost.sum() / world + cost.max()
    with pytest.raises(ValueError):
        direction_blocks(cost, p.n_dirs + 1)


def test_direction_cost_uses_the_oracle_geometry():
    """The host-side cost model (n_sub + 1 per direction) is the oracle's sub-segment count,
    the one the CUDA setup (csrc/lattice.cu: setup_lattice) computes with the same formula."""
    sys.path.insert(0, ROOT)
    from oracle import lattice as OL
    from paper_2602_21958_b200 import lattice as L
    from paper_2602_21958_b200.sharding import lattice_direction_cost

    for ny in (1, 6):
        p = L.lattice_problem(7, ny, 5, 8, 12, 3, layout="moments")
        d = OL.desc_from_lattice_problem(p)
        n_sub = np.array([OL.direction_geometry(d, a)[3] for a in range(p.n_dirs)])
        np.testing.assert_array_equal(lattice_direction_cost(p), n_sub + 1)


class OracleLatticeSpaceOps(OracleLatticeShardOps):
    def apply_with_moments_nodes(self, u_b, m_b, node0, node1):
        import torch

        d = self.d
        nodes = node1 - node0
        Rm = self.OL.redistribute(d, np.asarray(m_b, dtype=float).reshape(nodes, d.n_mom, d.n_freq))
        return torch.from_numpy(np.asarray(u_b, dtype=float) - Rm.reshape(-1))


def _space_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist

    from oracle import lattice as OL
    from paper_2602_21958_b200.sharding import LatticeSpaceShardedOperator, sharded_gmres

    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = _problem()
    op = LatticeSpaceShardedOperator(p, ops_factory=OracleLatticeSpaceOps)
    u = torch.from_numpy(np.random.default_rng(3).standard_normal(p.n_total))
    y_b = op(op.local_slice(u))
    d = OL.desc_from_lattice_problem(p)
    b = torch.from_numpy(OL.build_rhs(d, "moments"))
    x_b, its, conv, hist, tr = sharded_gmres(op, op.local_slice(b).clone(), rel_tol=1e-9, max_iter=300)
    q.put((rank, (op.node0, op.node1), y_b.numpy().tolist(), its, x_b.numpy().tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
@pytest.mark.parametrize("world", [2, 3])
def test_space_sharded_ranks_reproduce_the_operator_and_gmres(world):
    """Krylov vectors sharded by layers (all-gather u, direction-block transfer, reduce-scatter of
    the moments by space, finish on the rank's layers): the blocks of all ranks form apply_A, and
    sharded_gmres on the blocks takes the single-process GMRES path (3 ranks: uneven blocks)."""
    from oracle import lattice as OL
    from oracle import rt_oracle as ro

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 30100 + world * 37 + os.getpid() % 800
    procs = [ctx.Process(target=_space_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    out = sorted(q.get(timeout=280) for _ in procs)
    for pr in procs:
        pr.join(timeout=30)
    assert all(pr.exitcode == 0 for pr in procs)
    p = _problem()
    d = OL.desc_from_lattice_problem(p)
    u = np.random.default_rng(3).standard_normal(p.n_total)
    ref = OL.apply_A_moments(d, u)
    y = np.concatenate([np.asarray(o[2]) for o in out])
    assert [o[1] for o in out][0][0] == 0 and out[-1][1][1] == p.n_space
    assert np.linalg.norm(y - ref) <= 1e-13 * np.linalg.norm(ref)
    b = OL.build_rhs(d, "moments")
    single = ro.gmres(lambda v: OL.apply_A_moments(d, v), b, rel_tol=1e-9, max_iter=300)
    assert len({o[3] for o in out}) == 1 and abs(out[0][3] - single.iterations) <= 1
    x = np.concatenate([np.asarray(o[4]) for o in out])
    sol = np.asarray(single.solution)
    assert np.linalg.norm(x - sol) <= 1e-7 * np.linalg.norm(sol)
