"""Multi-rank host logic of the sharded loop (paper_2212_11506_b200/dist.py)
on CPU with gloo, world sizes 2 and 3.

Each rank computes its shard of the forces with the CPU oracle (the stand-in
for the CUDA kernels here), the shards are exchanged with all_gather_into_
tensor exactly as Shard lays them out, and the assembled gradient and Z
must equal the single-process result bit for bit -- the property that makes
the GPU trajectory independent of the GPU count.
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2212_11506_b200.dist import POINTS_PER_PARTIAL, ShardPlan  # noqa: E402


def fixed_sum(x):
    """Host mirror of the device fixed_sum: 32 lane-strided sequential
    partials, then an xor butterfly."""
    lanes = np.zeros(32)
    for i, v in enumerate(x):
        lanes[i % 32] = lanes[i % 32] + v
    for o in (16, 8, 4, 2, 1):
        lanes = np.array([lanes[l] + lanes[l ^ o] for l in range(32)])
    return lanes[0]


def problem():
    from oracle import oracle as o
    rng = np.random.default_rng(5)
    n = 2000
    centres = rng.uniform(-5, 5, (3, 6))
    x = (centres[rng.integers(0, 3, n)] + rng.standard_normal((n, 6))).astype(np.float32)
    idx, sqd = o.knn_exact(x, 20)
    _, cond = o.calibrate_perplexity(sqd, 7.0)
    ro, co, va = o.symmetrize(idx, cond)
    y = (rng.standard_normal((n, 2)) * 2).astype(np.float32)
    return y, ro, co, va


def shard_forces(o, y, ro, co, va, plan):
    """What one rank's kernels produce: attr rows, sorted-order rep, Z
    partials of its POINTS_PER_PARTIAL-point blocks."""
    n = y.shape[0]
    t = o.build_tree(y, code_bits=32)          # replicated tree
    a0, a1 = o.attractive(ro, co, va, y)
    r0, r1, zp, _ = o.repulsive_bh(t, y, 0.5)
    lo, hi = plan.mine
    attr = np.zeros((plan.chunk, 2), np.float32)
    attr[:hi - lo] = np.column_stack([a0, a1])[lo:hi]
    rep = np.zeros((plan.chunk, 2), np.float32)
    rep[:hi - lo] = np.column_stack([r0, r1])[t.order[lo:hi]]
    z = np.zeros(plan.partials_per_rank)
    zs = zp[t.order]
    for b in range(plan.partials_per_rank):
        s, e = lo + b * POINTS_PER_PARTIAL, min(hi, lo + (b + 1) * POINTS_PER_PARTIAL)
        if s < e:
            z[b] = np.sum(zs[s:e])
    return attr, rep, z, t.order


def worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as o
        o.build()
        y, ro, co, va = problem()
        n = y.shape[0]
        plan = ShardPlan(n, world, rank)
        attr, rep, z, order = shard_forces(o, y, ro, co, va, plan)
        A = torch.zeros((plan.gathered_len(), 2))
        R = torch.zeros((plan.gathered_len(), 2))
        Z = torch.zeros(world * plan.partials_per_rank, dtype=torch.float64)
        dist.all_gather_into_tensor(A, torch.from_numpy(attr))
        dist.all_gather_into_tensor(R, torch.from_numpy(rep))
        dist.all_gather_into_tensor(Z, torch.from_numpy(z))
        rank_of = np.empty(n, np.int64)
        rank_of[order] = np.arange(n)
        attr_full = A.numpy()[:n]
        rep_full = R.numpy()[rank_of]
        zt = fixed_sum(Z.numpy())
        if rank == 0:
            q.put((attr_full, rep_full, zt))
    finally:
        dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_plan_ranges_cover_and_align():
    for n in (1, 255, 256, 1000, 70_000, 1_300_000):
        for world in (1, 2, 3, 4, 8):
            ranges = [ShardPlan(n, world, r).mine for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == n
            for (a, b), (c, d) in zip(ranges, ranges[1:]):
                assert b == c
            chunk = ShardPlan(n, world, 0).chunk
            assert chunk % POINTS_PER_PARTIAL == 0
            for a, _ in ranges:
                assert a % POINTS_PER_PARTIAL == 0 or a == n


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_forces_equal_single_process(oracle, world):
    y, ro, co, va = problem()
    n = y.shape[0]
    attr1, rep1, z1, order1 = shard_forces(oracle, y, ro, co, va,
                                           ShardPlan(n, 1, 0))
    rank_of = np.empty(n, np.int64)
    rank_of[order1] = np.arange(n)
    ref_attr, ref_rep, ref_z = attr1[:n], rep1[rank_of], fixed_sum(z1)
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    mp.start_processes(worker, args=(world, free_port(), q), nprocs=world,
                       join=True, start_method="spawn")
    attr, rep, z = q.get()
    np.testing.assert_array_equal(attr, ref_attr)
    np.testing.assert_array_equal(rep, ref_rep)
    assert z == ref_z  # bitwise: Z independent of the world size
