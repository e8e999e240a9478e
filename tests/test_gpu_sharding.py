"""Device halves of the direction-sharded operator on one GPU: the shards' partial moments
(rtk_partial_moments) summed by hand stand in for the all-reduce, then every shard's
rtk_apply_A_with_moments; the reassembled vector must equal the single-GPU operator and
the oracle (1e-11)."""
import numpy as np
import pytest
import torch

import paper_2602_21958_b200 as P
from paper_2602_21958_b200 import configs
from paper_2602_21958_b200.sharding import ShardedOperator
from oracle import rt_oracle as ro
from tests._problems import rel_l2

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("shape", [(100, 16, 31), (300, 16, 128), (2000, 64, 512)])
def test_sharded_matvec_equals_full_operator(world, shape):
    ns, na, nf = shape
    p = configs.slab_problem(2, n_space=ns, n_angles=na, n_freq=nf)
    x = torch.from_numpy(np.random.default_rng(ns).standard_normal(p.n_total)).cuda()
    ops = [ShardedOperator(p, rank=r, world=world, all_reduce=lambda t: t) for r in range(world)]
    locals_ = [op.local_slice(x).contiguous() for op in ops]
    m = sum(op.ops.partial_moments(xl) for op, xl in zip(ops, locals_))   # the all-reduce
    g = p.grid
    y = torch.empty(g.n_space, g.n_angles, g.n_freq, dtype=torch.float64, device="cuda")
    for op, xl in zip(ops, locals_):
        a0, a1 = int(op.angles[0]), int(op.angles[-1]) + 1
        y[:, a0:a1, :] = op.ops.apply_with_moments(xl, m.clone()).reshape(g.n_space, a1 - a0, g.n_freq)
    y = y.reshape(-1)
    full = P.apply_A(p, x)
    assert rel_l2(y.cpu().numpy(), full.cpu().numpy()) <= 1e-12
    if ns <= 300:
        assert rel_l2(y.cpu().numpy(), ro.apply_A(ro.desc_from_problem(p), x.cpu().numpy())) <= 1e-11


def test_sharded_gmres_single_rank_matches_native_gmres():
    """sharded_gmres with the native device halves (one rank, identity all-reduce) reproduces the
    native GMRES: iterations +-1, history prefix, solution 1e-7."""
    from paper_2602_21958_b200.sharding import sharded_gmres

    p = configs.slab_problem(1)
    op = ShardedOperator(p, rank=0, world=1, all_reduce=lambda t: t)
    b = P.build_rhs(p, device=True)
    x, its, conv, hist, _ = sharded_gmres(op, b, rel_tol=1e-8, max_iter=300)
    rep = P.gmres(p, b, P.SolveConfig(rel_tol=1e-8, max_iter=300))
    assert conv and rep.converged and abs(its - rep.iterations) <= 1
    np.testing.assert_allclose(hist[:30], rep.residual_history[:30], rtol=1e-9)
    assert rel_l2(x.cpu().numpy(), rep.solution.cpu().numpy()) <= 1e-7


# ---------------- lattice problems, moment layout (configs 4-5) ----------------

@pytest.mark.parametrize("world", [2, 3, 5])
@pytest.mark.parametrize("fs", ["ie", "exp_linear", "exp_parabolic"])
def test_lattice_sharded_matvec_equals_full_operator(world, fs):
    """rtk_lattice_partial_moments over a partition of the directions, summed (the all-reduce),
    then rtk_lattice_apply_with_moments: equals rtk_apply_A and the oracle."""
    from oracle import lattice as OL
    from paper_2602_21958_b200 import lattice as L
    from paper_2602_21958_b200.sharding import LatticeShardedOperator

    p = L.lattice_problem(7, 6, 6, 8, 8, 4, corr_len=2.0, seed=21, layout="moments", formal_solver=fs,
                          characteristics="hybrid")
    u = torch.from_numpy(np.random.default_rng(world).standard_normal(p.n_total)).cuda()
    ops = [LatticeShardedOperator(p, rank=r, world=world, all_reduce=lambda t: t) for r in range(world)]
    m = sum(op.ops.partial_moments(u) for op in ops)
    ys = [op.ops.apply_with_moments(u, m.clone()) for op in ops]
    full = P.apply_A(p, u)
    for y in ys:
        assert rel_l2(y.cpu().numpy(), full.cpu().numpy()) <= 1e-12
    ref = OL.apply_A(OL.desc_from_lattice_problem(p), "moments", u.cpu().numpy())
    assert rel_l2(ys[0].cpu().numpy(), ref) <= 1e-11


def test_lattice_sharded_cfg4_full_size_equals_full_operator():
    """cfg4 size (64^3, 128 directions, 31 nu): two direction blocks reassemble the operator."""
    from paper_2602_21958_b200 import lattice as L
    from paper_2602_21958_b200.sharding import LatticeShardedOperator

    p = L.lattice_problem(64, 64, 64, 8, 16, 31, corr_len=8.0, seed=21962, layout="moments")
    u = torch.randn(p.n_total, dtype=torch.float64, device="cuda")
    ops = [LatticeShardedOperator(p, rank=r, world=2, all_reduce=lambda t: t) for r in range(2)]
    m = ops[0].ops.partial_moments(u) + ops[1].ops.partial_moments(u)
    y = ops[1].ops.apply_with_moments(u, m)
    full = P.apply_A(p, u)
    assert float(torch.linalg.vector_norm(y - full) / torch.linalg.vector_norm(full)) <= 1e-12


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("fs", ["ie", "exp_linear"])
def test_lattice_space_sharded_blocks_form_the_operator(world, fs):
    """The space-sharded lattice operator's device halves, ranks emulated in lockstep on one GPU:
    rtk_lattice_partial_moments over each rank's direction block on the gathered u, summed and
    split by layer blocks (the reduce-scatter), then rtk_lattice_apply_with_moments_nodes per
    block -- the concatenated blocks equal rtk_apply_A."""
    from paper_2602_21958_b200 import lattice as L
    from paper_2602_21958_b200.sharding import LatticeSpaceShardedOperator

    p = L.lattice_problem(7, 6, 7, 8, 8, 5, corr_len=2.0, seed=23, layout="moments", formal_solver=fs,
                          characteristics="hybrid")
    u = torch.from_numpy(np.random.default_rng(world).standard_normal(p.n_total)).cuda()
    ops = [LatticeSpaceShardedOperator(p, rank=r, world=world, all_reduce=lambda t: t) for r in range(world)]
    m = sum(op.ops.partial_moments(u) for op in ops)
    ys = []
    for op in ops:
        m_b = op.local_slice(m).contiguous()
        ys.append(op.ops.apply_with_moments_nodes(op.local_slice(u).contiguous(), m_b, op.node0, op.node1))
    y = torch.cat(ys)
    full = P.apply_A(p, u)
    assert float(torch.linalg.vector_norm(y - full) / torch.linalg.vector_norm(full)) <= 1e-12
