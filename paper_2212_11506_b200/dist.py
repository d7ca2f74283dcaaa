"""Multi-GPU data parallelism for the BH t-SNE loop.

One process per GPU (torchrun), NCCL over NVLink/NVSwitch.  Each rank keeps
the full Y replicated and rebuilds the small 2-D tree redundantly; the force
work is sharded contiguously:

* repulsion: sorted (Morton-order) positions [t0, t1) of rank r, so a rank's
  warps walk coherent paths;
* attraction: CSR rows [r0, r1) (point ids).

One exchange per iteration: an all-gather of the attractive rows, the
sorted-order repulsive forces and the per-128-point Z partials.  Every rank
then runs the (cheap, elementwise) update for all N points on identical
inputs, so Y stays replicated without a separate Y all-gather.  In the
untimed fast path the attractive rows and their all-gather run on a side
stream (with their own communicator) under the replicated tree build, so
only the repulsive exchange remains on the critical path.  Ranges are
multiples of 128 points, so the gathered Z partials are exactly the blocks
a single GPU produces and Z -- hence the whole trajectory -- is bitwise
independent of the GPU count.

``ShardPlan`` is the pure host logic (ranges, buffer layout, assembly) and
is exercised with gloo on CPU in tests/test_dist.py; ``Shard`` binds it to
the CUDA engine.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

POINTS_PER_PARTIAL = 128  # BH_REP_POINTS_PER_PARTIAL (include/bhtsne_b200.h)


@dataclass(frozen=True)
class ShardPlan:
    n: int
    world: int
    rank: int

    @property
    def chunk(self) -> int:
        """Points per rank, a multiple of POINTS_PER_PARTIAL."""
        per = math.ceil(self.n / self.world)
        return math.ceil(per / POINTS_PER_PARTIAL) * POINTS_PER_PARTIAL

    def range_of(self, r: int) -> tuple:
        lo = min(self.n, r * self.chunk)
        return lo, min(self.n, lo + self.chunk)

    @property
    def mine(self) -> tuple:
        return self.range_of(self.rank)

    @property
    def partials_per_rank(self) -> int:
        return self.chunk // POINTS_PER_PARTIAL

    @property
    def total_partials(self) -> int:
        return math.ceil(self.n / POINTS_PER_PARTIAL)

    def gathered_len(self) -> int:
        return self.world * self.chunk


class Shard:
    """Engine hooks: sharded forces + one NCCL all-gather per iteration."""

    def __init__(self, rank: int, world: int, group=None):
        self.rank, self.world, self.group = rank, world, group
        self.side_group = None

    def attach(self, eng):
        import torch
        import torch.distributed as dist

        from .quadtree import TreeArrays
        self.plan = ShardPlan(eng.n, self.world, self.rank)
        pl = self.plan
        dev = eng.dev
        f32 = dict(dtype=eng.dtype, device=dev)  # the run precision
        self.attr_send = torch.zeros((pl.chunk, 2), **f32)
        self.rep_send = torch.zeros((pl.chunk, 2), **f32)
        self.z_send = torch.zeros(pl.partials_per_rank, dtype=torch.float64,
                                  device=dev)
        self.attr_all = torch.zeros((pl.gathered_len(), 2), **f32)
        self.rep_all = torch.zeros((pl.gathered_len(), 2), **f32)
        self.z_all = torch.zeros(self.world * pl.partials_per_rank,
                                 dtype=torch.float64, device=dev)
        # the tree must publish rank[id] = sorted position for the update
        self.rank_of = torch.zeros(eng.n, dtype=torch.int32, device=dev)
        eng.tree.struct.rank = self.rank_of.data_ptr()
        eng.attr = self.attr_all[:eng.n]
        # a second communicator for the side-stream attr gather (collectives
        # of one communicator must not run concurrently on two streams)
        ranks = (list(range(self.world)) if self.group is None
                 else dist.get_process_group_ranks(self.group))
        self.side_group = dist.new_group(ranks=ranks)
        # warm the communicators outside any graph capture
        self._gather()
        self._gather_attr(self.side_group)
        torch.cuda.synchronize()

    def _gather_attr(self, group):
        import torch.distributed as dist
        dist.all_gather_into_tensor(self.attr_all, self.attr_send, group=group)

    def _gather_rep(self):
        import torch.distributed as dist
        g = self.group
        dist.all_gather_into_tensor(self.rep_all, self.rep_send, group=g)
        dist.all_gather_into_tensor(self.z_all, self.z_send, group=g)

    def _gather(self):
        self._gather_attr(self.group)
        self._gather_rep()

    def attractive(self, eng, st):
        """This rank's CSR rows [r0, r1) into attr_send."""
        from ._lib import call, ptr
        import ctypes as C
        r0, r1 = self.plan.mine
        # attr[row] for rows [r0, r1) lands at attr_send[row - r0]
        base = C.c_void_p(self.attr_send.data_ptr() - eng.pt_bytes * r0)
        call(eng.fn("bh_attractive"), ptr(eng.rp), ptr(eng.col), ptr(eng.val),
             eng.n, 1, ptr(eng.y), r0, r1, 1.0, ptr(eng.sched), base, st)

    def attractive_side(self, eng):
        """Attractive rows + their all-gather on the current (side) stream,
        with the side communicator."""
        from ._lib import stream
        self.attractive(eng, stream())
        self._gather_attr(self.side_group)

    def repulsive(self, eng, rec, st):
        """Sorted positions [r0, r1), then the rep / Z exchange and Z."""
        from ._lib import call, ptr
        r0, r1 = self.plan.mine
        call(eng.fn("bh_repulsive"), eng.tree.sref(), ptr(eng.bounds),
             eng.theta, None, r0, r1, 1, ptr(self.rep_send), None,
             ptr(self.z_send), None, None, ptr(eng.ws_rep),
             eng.ws_rep.numel(), st)
        rec(4)
        self._gather_rep()
        call("bh_sum_partials", ptr(self.z_all), self.z_all.numel(),
             ptr(eng.z_dev), st)
        rec(5)
        return self.rep_all, self.rank_of

    def forces(self, eng, rec, st):
        """Sequential: attractive, repulsive, then all three exchanges."""
        self.attractive(eng, st)
        rec(3)
        self._gather_attr(self.group)
        return self.repulsive(eng, rec, st)

    @staticmethod
    def comm_time(ev) -> float:
        return ev[4].elapsed_time(ev[5]) * 1e-3
