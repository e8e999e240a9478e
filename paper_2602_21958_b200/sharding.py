"""Direction-sharded (I - Lambda Sigma) for several GPUs.

Lambda is independent per (direction, frequency) and Sigma couples
the directions only through the angular moments, so the operator
shards by direction with ONE exchange per matvec: every rank holds all of space
x all frequencies x its block of directions, computes the partial moments of
its slice of x, the partial moments are summed across ranks (one all-reduce of
n_space x n_mom x N_nu values: 16 MB at cfg2), and each rank redistributes the
summed moments (replicated DMMA GEMM) and sweeps its own rays.

    op = ShardedOperator(problem)              # inside torch.distributed, NCCL on GPUs
    y_local = op(x_local)                      # x_local = op.local_slice(x)

The local pieces run through the C ABI (rtk_partial_moments /
rtk_apply_A_with_moments); the exchange is torch.distributed.all_reduce.
`ops_factory` / `all_reduce` are injectable so the host logic is testable on
CPU ranks (tests/test_sharding.py, gloo).  Slab problems, intensity layout;
lattice problems in the moment layout: LatticeShardedOperator below.
"""

from __future__ import annotations

import numpy as np

from paper_2602_21958_b200 import _device, _native
from paper_2602_21958_b200.grid import Grid
from paper_2602_21958_b200.operator import RTProblem
from paper_2602_21958_b200.scattering import ScatteringOperator, separable_form
from paper_2602_21958_b200.transfer import build_transfer


def angle_block(n_angles: int, rank: int, world: int) -> np.ndarray:
    """Directions of `rank`: a contiguous, balanced block of the angle index range."""
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of size {world}")
    if world > n_angles:
        raise ValueError(f"cannot shard {n_angles} directions over {world} ranks")
    lo = (n_angles * rank) // world
    hi = (n_angles * (rank + 1)) // world
    return np.arange(lo, hi)


def shard_problem(problem: RTProblem, rank: int, world: int):
    """(local problem on this rank's directions, their global indices).  The local grid keeps
    the global quadrature weights, so partial moments add up to the global ones."""
    if problem.layout != "intensity":
        raise ValueError("direction sharding needs the intensity layout")
    g = problem.grid
    sel = angle_block(g.n_angles, rank, world)
    grid = Grid(g.t_nodes, g.mu_nodes[sel], g.angular_weights[sel], g.nu_nodes, g.frequency_weights, g.profile)
    rays = (sel[:, None] * g.n_freq + np.arange(g.n_freq)[None, :]).reshape(-1)
    gamma = np.ascontiguousarray(np.asarray(problem.scattering.gamma_table).reshape(g.n_space, g.n_rays)[:, rays])
    scat = ScatteringOperator(grid, problem.scattering.kernel, gamma)
    tr = build_transfer(grid, 0.0, 0.0, formal_solver=problem.transfer.formal_solver)
    tr.inflow = np.asarray(problem.transfer.inflow)[rays]
    thermal = np.asarray(problem.thermal).reshape(g.n_space, g.n_rays)[:, rays].reshape(-1)
    desc = dict(problem.descriptor)
    desc.update({"shard": f"{rank}/{world}", "angles": [int(sel[0]), int(sel[-1]) + 1]})
    return RTProblem(grid, tr, scat, thermal=thermal, descriptor=desc), sel


class NativeShardOps:
    """The device halves of a sharded matvec on this rank's local problem."""

    def __init__(self, local: RTProblem):
        self.local = local
        self.n = local.n_total
        g = local.grid
        self.n_m = g.n_space * separable_form(local.scattering.kernel, g)[0].shape[0] * g.n_freq

    def partial_moments(self, x):
        h = self.local.device()
        m = _device.empty(self.n_m)
        _native.check(_native.lib().rtk_partial_moments(h.h, _device.ptr(x), _device.ptr(m), self.n_m,
                                                        _device.stream_ptr()))
        return m

    def apply_with_moments(self, x, m):
        h = self.local.device()
        y = _device.empty(self.n)
        _native.check(_native.lib().rtk_apply_A_with_moments(h.h, _device.ptr(x), _device.ptr(m), self.n_m,
                                                             _device.ptr(y), self.n, _device.stream_ptr()))
        return y


def _dist_all_reduce(t, group=None):
    import torch.distributed as dist

    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


class ShardedOperator:
    """y_local = (I - Lambda Sigma) x restricted to this rank's rays (see module docstring)."""

    def __init__(self, problem: RTProblem, rank: int = None, world: int = None, group=None,
                 ops_factory=NativeShardOps, all_reduce=None):
        if rank is None or world is None:
            import torch.distributed as dist

            rank = dist.get_rank(group) if rank is None else rank
            world = dist.get_world_size(group) if world is None else world
        self.problem = problem
        self.rank, self.world = rank, world
        self.local, self.angles = shard_problem(problem, rank, world)
        self.ops = ops_factory(self.local)
        self._all_reduce = all_reduce or (lambda t: _dist_all_reduce(t, group))

    def local_slice(self, x):
        """This rank's part of a global space-major vector (n_space x local directions x N_nu)."""
        g = self.problem.grid
        a0, a1 = int(self.angles[0]), int(self.angles[-1]) + 1
        return x.reshape(g.n_space, g.n_angles, g.n_freq)[:, a0:a1, :].reshape(-1)

    def __call__(self, x_local):
        m = self.ops.partial_moments(x_local)
        m = self._all_reduce(m)
        return self.ops.apply_with_moments(x_local, m)


# ---------------------------------------------------------------------------
# Multi-D lattice problems in the moment layout (configs 4-5)
#
# The unknown u (redistributed dipole moments, 4.1 GB at cfg5) is REPLICATED on every rank;
# rank r transfers only its block of directions [a0, a1) and produces partial angular moments;
# one all-reduce of n_space x n_mom x N_nu values sums them, and every rank finishes
# y = u - R_w m.  All ranks then hold identical y (the all-reduce delivers the same sum to
# every rank), so any solver can run redundantly on the replicated vectors -- including the
# native GMRES through a callable.  Directions are split by transfer cost (sub-segments per
# layer step), not by count: grazing directions cost several times a steep one.


def lattice_direction_cost(problem) -> np.ndarray:
    """Relative transfer cost of each direction: n_sub + 1 sub-node samples per layer step
    (the geometry of oracle/lattice.py: n_sub = ceil(max(|sx|, |sy|)))."""
    om = np.asarray(problem.omega, dtype=float)
    sx = np.abs(om[:, 0] * problem.dz / (np.abs(om[:, 2]) * problem.dx))
    sy = np.abs(om[:, 1] * problem.dz / (np.abs(om[:, 2]) * problem.dy)) if problem.ny > 1 else 0.0 * sx
    n_sub = np.maximum(1, np.ceil(np.maximum(sx, sy) - 1e-12)).astype(int)
    return n_sub + 1.0


def direction_blocks(cost: np.ndarray, world: int):
    """Contiguous direction ranges [(a0, a1)] with balanced total cost, one per rank."""
    n = cost.size
    if world > n:
        raise ValueError(f"cannot shard {n} directions over {world} ranks")
    csum = np.concatenate([[0.0], np.cumsum(cost)])
    bounds = [0]
    for r in range(1, world):
        target = csum[-1] * r / world
        b = int(np.searchsorted(csum, target))
        b = min(max(b, bounds[-1] + 1), n - (world - r))
        bounds.append(b)
    bounds.append(n)
    return [(bounds[r], bounds[r + 1]) for r in range(world)]


class NativeLatticeShardOps:
    """Device halves of a direction-sharded lattice matvec (rtk_lattice_partial_moments /
    rtk_lattice_apply_with_moments)."""

    def __init__(self, problem, a0: int, a1: int):
        self.problem, self.a0, self.a1 = problem, a0, a1
        self.n = problem.n_total

    def partial_moments(self, u):
        h = self.problem.device()
        m = _device.empty(self.n)
        _native.check(_native.lib().rtk_lattice_partial_moments(h.h, _device.ptr(u), _device.ptr(m), self.n,
                                                                self.a0, self.a1, _device.stream_ptr()))
        return m

    def apply_with_moments(self, u, m):
        h = self.problem.device()
        y = _device.empty(self.n)
        _native.check(_native.lib().rtk_lattice_apply_with_moments(h.h, _device.ptr(u), _device.ptr(m), self.n,
                                                                   _device.ptr(y), self.n, _device.stream_ptr()))
        return y


class LatticeShardedOperator:
    """y = u - R_w M Lambda S(u) with the directions split over the ranks (see above); u and y
    are full, replicated vectors."""

    def __init__(self, problem, rank: int = None, world: int = None, group=None,
                 ops_factory=NativeLatticeShardOps, all_reduce=None):
        if getattr(problem, "layout", None) != "moments":
            raise ValueError("lattice direction sharding needs the moment layout")
        if rank is None or world is None:
            import torch.distributed as dist

            rank = dist.get_rank(group) if rank is None else rank
            world = dist.get_world_size(group) if world is None else world
        self.problem = problem
        self.rank, self.world = rank, world
        self.blocks = direction_blocks(lattice_direction_cost(problem), world)
        self.a0, self.a1 = self.blocks[rank]
        self.ops = ops_factory(problem, self.a0, self.a1)
        self._all_reduce = all_reduce or (lambda t: _dist_all_reduce(t, group))

    def __call__(self, u):
        m = self.ops.partial_moments(u)
        m = self._all_reduce(m)
        return self.ops.apply_with_moments(u, m)


# ---------------------------------------------------------------------------
# Lattice problems, moment layout, Krylov vectors sharded by SPACE
#
# Rank r owns a contiguous block of layers of u (its Krylov vectors are that block only) and
# a cost-balanced block of directions.  One matvec:
#   all-gather u (every rank needs the source on all layers its directions cross),
#   transfer of the rank's directions -> partial moments on ALL of space,
#   reduce-scatter by space -> the summed moments of the rank's layers,
#   y_b = u_b - R_w m_b on the rank's layers (rtk_lattice_apply_with_moments_nodes).
# The collective volume equals the all-reduce of the replicated variant (an all-reduce is a
# reduce-scatter plus an all-gather), but the Krylov basis, the CGS2 passes and the
# redistribution GEMM are divided by the world size instead of replicated (cfg5: 21 basis
# vectors x 4.1 GB on every GPU replicated, 4.1 / W GB each sharded).


def layer_blocks(nz: int, world: int):
    """Contiguous layer ranges [(k0, k1)], sizes differing by at most one."""
    if world > nz:
        raise ValueError(f"cannot shard {nz} layers over {world} ranks")
    return [((nz * r) // world, (nz * (r + 1)) // world) for r in range(world)]


class NativeLatticeSpaceOps(NativeLatticeShardOps):
    """Device halves of the space-sharded lattice matvec."""

    def apply_with_moments_nodes(self, u_b, m_b, node0: int, node1: int):
        h = self.problem.device()
        y = _device.empty(u_b.numel())
        _native.check(_native.lib().rtk_lattice_apply_with_moments_nodes(
            h.h, _device.ptr(u_b), _device.ptr(m_b), node0, node1, _device.ptr(y), _device.stream_ptr()))
        return y


def _dist_all_gather(t, group=None):
    import torch
    import torch.distributed as dist

    out = torch.empty(t.numel() * dist.get_world_size(group), dtype=t.dtype, device=t.device)
    dist.all_gather_into_tensor(out, t, group=group)
    return out


def _dist_reduce_scatter(t, group=None):
    import torch
    import torch.distributed as dist

    out = torch.empty(t.numel() // dist.get_world_size(group), dtype=t.dtype, device=t.device)
    dist.reduce_scatter_tensor(out, t, op=dist.ReduceOp.SUM, group=group)
    return out


class LatticeSpaceShardedOperator:
    """y_b = (u - R_w M Lambda S(u))_b on this rank's layer block b (see above).  Vectors are
    local blocks; uneven blocks are padded to the largest for the collectives."""

    def __init__(self, problem, rank: int = None, world: int = None, group=None,
                 ops_factory=NativeLatticeSpaceOps, all_reduce=None, all_gather=None, reduce_scatter=None):
        if getattr(problem, "layout", None) != "moments":
            raise ValueError("lattice sharding needs the moment layout")
        if rank is None or world is None:
            import torch.distributed as dist

            rank = dist.get_rank(group) if rank is None else rank
            world = dist.get_world_size(group) if world is None else world
        self.problem = problem
        self.rank, self.world = rank, world
        self.a0, self.a1 = direction_blocks(lattice_direction_cost(problem), world)[rank]
        self.layers = layer_blocks(problem.nz, world)
        nxy = problem.nx * problem.ny
        self.per_node = problem.n_mom * problem.n_freq
        self.nodes = [(k0 * nxy, k1 * nxy) for k0, k1 in self.layers]
        self.node0, self.node1 = self.nodes[rank]
        self.pad = max(n1 - n0 for n0, n1 in self.nodes) * self.per_node
        self.ops = ops_factory(problem, self.a0, self.a1)
        self._all_reduce = all_reduce or (lambda t: _dist_all_reduce(t, group))
        self._all_gather = all_gather or (lambda t: _dist_all_gather(t, group))
        self._reduce_scatter = reduce_scatter or (lambda t: _dist_reduce_scatter(t, group))

    def local_slice(self, u):
        return u[self.node0 * self.per_node:self.node1 * self.per_node]

    def _padded(self, v, lo, hi):
        import torch

        out = torch.zeros(self.pad, dtype=v.dtype, device=v.device)
        out[:(hi - lo) * self.per_node] = v
        return out

    def gather(self, u_b):
        """The full vector from the blocks of all ranks."""
        g = self._all_gather(self._padded(u_b, self.node0, self.node1))
        import torch

        return torch.cat([g[r * self.pad:r * self.pad + (n1 - n0) * self.per_node]
                          for r, (n0, n1) in enumerate(self.nodes)])

    def scatter_sum(self, m):
        """Sum over ranks of m, this rank's block (reduce-scatter by space)."""
        import torch

        blocks = [self._padded(m[n0 * self.per_node:n1 * self.per_node], n0, n1) for n0, n1 in self.nodes]
        part = self._reduce_scatter(torch.cat(blocks))
        return part[:(self.node1 - self.node0) * self.per_node]

    def __call__(self, u_b):
        u = self.gather(u_b)
        m = self.ops.partial_moments(u)
        m_b = self.scatter_sum(m)
        return self.ops.apply_with_moments_nodes(u_b, m_b.contiguous(), self.node0, self.node1)


def sharded_gmres(op: ShardedOperator, b_local, rel_tol: float = 1e-12, max_iter: int = 1000, restart: int = None):
    """GMRES on direction-sharded vectors (R/krylov.py:56-158 control flow: x0 = 0, Givens least
    squares, restart, breakdown below 1e-14 ||b||, 10 rel_tol true-residual guard).  Every rank
    holds its slice of the Krylov vectors; the dots are local products plus one all-reduce, so
    all ranks see the same scalars and take the same decisions.  Arnoldi is CGS2 (as the native
    solver).  Returns (x_local, iterations, converged, residual history, true residual)."""
    import torch

    def gdot(u, v):
        t = torch.dot(u, v).reshape(1)
        return float(op._all_reduce(t)[0])

    def gnorm(u):
        return gdot(u, u) ** 0.5

    b = b_local
    b_norm = gnorm(b)
    hist = []
    if b_norm == 0.0:
        return torch.zeros_like(b), 0, True, [0.0], 0.0
    x = torch.zeros_like(b)
    r = b.clone()
    total = 0
    cycle = restart if restart is not None else max_iter
    while total < max_iter:
        beta = gnorm(r)
        if beta / b_norm <= rel_tol:
            hist.append(beta / b_norm)
            return x, max(total, 1), True, hist, beta / b_norm
        V = [r / beta]
        h_cols, cs, sn, g = [], [], [], [beta]
        breakdown = False
        steps = min(cycle, max_iter - total)
        j = 0
        while j < steps:
            w = op(V[j])
            Vm = torch.stack(V)                                        # (j+1, n_local)
            h1 = op._all_reduce(Vm @ w)
            w = w - Vm.t() @ h1
            h2 = op._all_reduce(Vm @ w)
            w = w - Vm.t() @ h2
            col = (h1 + h2).tolist()
            col.append(gnorm(w))
            breakdown = col[j + 1] < 1e-14 * b_norm
            if not breakdown:
                V.append(w / col[j + 1])
            for i in range(j):
                tmp = cs[i] * col[i] + sn[i] * col[i + 1]
                col[i + 1] = -sn[i] * col[i] + cs[i] * col[i + 1]
                col[i] = tmp
            denom = (col[j] ** 2 + col[j + 1] ** 2) ** 0.5
            cj = col[j] / denom if denom else 1.0
            sj = col[j + 1] / denom if denom else 0.0
            cs.append(cj)
            sn.append(sj)
            col[j] = denom
            h_cols.append(col[: j + 1])
            g.append(-sj * g[j])
            g[j] = cj * g[j]
            total += 1
            j += 1
            rel = abs(g[j]) / b_norm
            hist.append(rel)
            if rel <= rel_tol or breakdown:
                y = _solve_upper(h_cols, g[:j])
                cand = x + sum(yi * vi for yi, vi in zip(y, V))
                true_rel = gnorm(b - op(cand)) / b_norm
                if true_rel <= 10.0 * rel_tol:
                    if breakdown:
                        hist[-1] = true_rel
                    return cand, total, True, hist, true_rel
                if breakdown:
                    return cand, total, False, hist, true_rel
        y = _solve_upper(h_cols, g[:j])
        x = x + sum(yi * vi for yi, vi in zip(y, V))
        r = b - op(x)
    return x, total, False, hist, gnorm(r) / b_norm


def _solve_upper(h_cols, g):
    """Back substitution on the rotated Hessenberg columns (R/krylov.py:161-170)."""
    m = len(g)
    y = [0.0] * m
    for i in range(m - 1, -1, -1):
        s = g[i]
        for k in range(i + 1, m):
            s -= h_cols[k][i] * y[k]
        y[i] = s / h_cols[i][i]
    return y
