"""Multi-rank host logic of the sharded loop (paper_2212_11506_b200/dist.py)
on CPU with gloo, world sizes 2 and 3.

Each rank takes its cost-balanced share of the storage slots
(``balanced_cuts``, the host mirror of bh_partition), computes the forces of
its share with the CPU oracle (the stand-in for the CUDA kernels here),
writes its Z partials (one per 128 slots, zero outside the share), the
partials are all-reduced, the rank updates its own slots, packs them into a
cap-row send buffer and the shares are all-gathered and unpacked by the
cuts -- exactly the buffers and collectives of Shard.  The assembled Y and Z
must equal the single-process result bit for bit: the property that makes
the GPU trajectory independent of the GPU count.
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2212_11506_b200.dist import (POINTS_PER_PARTIAL, W_POINT,  # noqa: E402
                                        balanced_cuts, equal_share, share_cap)


def fixed_sum(x):
    """Host mirror of the device cta_fold (forces.cuh): 256 thread-strided
    sequential partials, an xor butterfly per warp, the 8 warps in order."""
    th = np.zeros(256)
    for i, v in enumerate(x):
        th[i % 256] = th[i % 256] + v
    tot = 0.0
    for w in range(8):
        lanes = th[32 * w:32 * (w + 1)].copy()
        for o in (16, 8, 4, 2, 1):
            lanes = np.array([lanes[l] + lanes[l ^ o] for l in range(32)])
        tot = tot + lanes[0]
    return tot


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


def step_parts(o, y, ro, co, va):
    """Per-point forces and per-128-slot Z partials of one iteration, and
    the elementwise update of every point (storage order = ids here)."""
    n = y.shape[0]
    t = o.build_tree(y, code_bits=32)          # replicated tree
    a0, a1 = o.attractive(ro, co, va, y)
    r0, r1, zp, _ = o.repulsive_bh(t, y, 0.5)
    nb = (n + POINTS_PER_PARTIAL - 1) // POINTS_PER_PARTIAL
    zblk = np.array([np.sum(zp[b * POINTS_PER_PARTIAL:(b + 1) * POINTS_PER_PARTIAL])
                     for b in range(nb)])
    return (a0, a1), (r0, r1), zblk


def updated(o, y, attr, rep, z):
    s = o.State(np.ascontiguousarray(y[:, 0]), np.ascontiguousarray(y[:, 1]),
                np.zeros(y.shape[0], np.float32), np.zeros(y.shape[0], np.float32),
                np.ones(y.shape[0], np.float32), np.ones(y.shape[0], np.float32))
    o.update(s, attr, rep, z, 0.5)
    return np.column_stack([s.y0, s.y1])


def worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as o
        o.build()
        y, ro, co, va = problem()
        n = y.shape[0]
        cap = share_cap(n, world)
        cuts = balanced_cuts(ro, n, world, cap=cap)
        lo, hi = int(cuts[rank]), int(cuts[rank + 1])
        attr, rep, zblk = step_parts(o, y, ro, co, va)
        # this rank's Z partials; the others' stay zero
        z = np.zeros_like(zblk)
        z[lo // POINTS_PER_PARTIAL:(hi + POINTS_PER_PARTIAL - 1) // POINTS_PER_PARTIAL] = \
            zblk[lo // POINTS_PER_PARTIAL:(hi + POINTS_PER_PARTIAL - 1) // POINTS_PER_PARTIAL]
        zt = torch.from_numpy(z)
        dist.all_reduce(zt)
        ztot = fixed_sum(zt.numpy())
        # the share's update, packed into the cap-row send buffer
        ynew = updated(o, y, attr, rep, ztot)
        send = np.zeros((cap, 2), np.float32)
        send[:hi - lo] = ynew[lo:hi]
        gbuf = torch.zeros((world * cap, 2))
        dist.all_gather_into_tensor(gbuf, torch.from_numpy(send))
        g = gbuf.numpy()
        y_all = np.empty_like(y)
        for r in range(world):  # bh_unpack_rows
            a, b = int(cuts[r]), int(cuts[r + 1])
            y_all[a:b] = g[r * cap:r * cap + (b - a)]
        if rank == 0:
            q.put((y_all, ztot))
    finally:
        dist.destroy_process_group()


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_balanced_cuts_cover_align_and_cap():
    rng = np.random.default_rng(1)
    for n in (1, 255, 256, 1000, 70_000, 1_300_000):
        lens = rng.integers(90, 400, n)
        lens[rng.integers(0, n, max(1, n // 50))] = 1200  # heavy rows
        rp = np.concatenate([[0], np.cumsum(lens)])
        for world in (1, 2, 3, 4, 8):
            cuts = balanced_cuts(rp, n, world)
            cap = share_cap(n, world)
            assert cuts[0] == 0 and cuts[-1] == n
            assert np.all(np.diff(cuts) >= 0)
            assert np.all(np.diff(cuts) <= cap)
            assert np.all((cuts[:-1] % POINTS_PER_PARTIAL == 0) | (cuts[:-1] == n))


def test_balanced_cuts_balance_cost():
    """Ranges follow the cost (W_POINT per point + row length), not the
    point count: a skewed row-length profile gets unequal point counts and
    near-equal costs."""
    n, world = 200_000, 8
    lens = np.where(np.arange(n) < n // 4, 1000, 90)  # heavy first quarter
    rp = np.concatenate([[0], np.cumsum(lens)])
    cuts = balanced_cuts(rp, n, world)
    cost = np.array([W_POINT * (cuts[r + 1] - cuts[r]) + rp[cuts[r + 1]] - rp[cuts[r]]
                     for r in range(world)])
    assert cost.max() / cost.mean() < 1.01
    assert len(set(np.diff(cuts).tolist())) > 1
    # a balanced range above the cap falls back to equal shares
    eq = balanced_cuts(rp, n, world, cap=equal_share(n, world))
    assert np.all(np.diff(eq)[:-1] == equal_share(n, world))


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_step_equals_single_process(oracle, world):
    y, ro, co, va = problem()
    attr, rep, zblk = step_parts(oracle, y, ro, co, va)
    ref_z = fixed_sum(zblk)
    ref_y = updated(oracle, y, attr, rep, ref_z)
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    mp.start_processes(worker, args=(world, free_port(), q), nprocs=world,
                       join=True, start_method="spawn")
    y_all, z = q.get()
    assert z == ref_z  # bitwise: Z independent of the world size
    np.testing.assert_array_equal(y_all, ref_y)
