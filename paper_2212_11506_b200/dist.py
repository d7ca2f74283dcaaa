"""Multi-GPU data parallelism for the BH t-SNE loop.

One process per GPU (torchrun), NCCL over NVLink/NVSwitch.  The reference
parallelises the same loop over CPU threads only (numba prange over points,
optimizer.py:273-286, forces.py:89); the partitioning here follows the
north star:

* every rank holds the full Y and rebuilds the small 2-D tree redundantly
  (Morton codes, sort, build, summarize of all N points);
* the points are the engine's storage slots (Morton order of the last
  relabel) and are sharded contiguously: rank r owns slots and CSR rows
  [c_r, c_{r+1}), cut at multiples of 128 and balanced by cost (a point
  weighs W_POINT CSR entries: the traversal against the sweep at C3);
* rank r computes the traversal of its slots and the attraction of its rows
  (one fused launch, the side-stream sweep included), then the Z partials
  -- one per 128 slots, zero outside the share -- are ALL-REDUCED (every
  element has exactly one non-zero term, so the sum is exact and Z is
  bitwise the single-GPU value), each rank updates its own slots, and the
  new Y of the shares is ALL-GATHERED (8 B per point in f32);
* the mean / bounds reduction then runs over the gathered Y in the
  single-GPU order (bh_step_finish), so the whole trajectory is bitwise
  independent of the GPU count.

Velocity and gains stay sharded; they are gathered only when the storage
order is renumbered (relabel, every relabel_every = 100 iterations) and at the end of a run.

``Shard`` binds this to the CUDA engine through a small collective
interface: ``NcclComm`` (torch.distributed, the product path, captured in
the engine's CUDA graphs) or ``LocalGroup`` (G ranks as threads of one
process on one GPU, their collectives done with stream-ordered copies -- the
multi-rank test of the real engine without G GPUs).  ``balanced_cuts`` is
the host mirror of bh_partition, checked against the device on the GPU and
used by the gloo tests on CPU.
"""

from __future__ import annotations

import math
import threading

import numpy as np

POINTS_PER_PARTIAL = 128  # BH_REP_POINTS_PER_PARTIAL (include/bhtsne_b200.h)
W_POINT = 270.0           # optimizer.W_POINT


def equal_share(n: int, world: int) -> int:
    per = math.ceil(n / world)
    return math.ceil(per / POINTS_PER_PARTIAL) * POINTS_PER_PARTIAL


def share_cap(n: int, world: int) -> int:
    """Rows per rank in the exchange buffers (optimizer.Engine.cap)."""
    if world == 1:
        return n
    a = POINTS_PER_PARTIAL
    return min(n, 2 * equal_share(n, world))


def balanced_cuts(row_ptr, n: int, world: int, w_point: float = W_POINT,
                  cap: int | None = None) -> np.ndarray:
    """Host mirror of bh_partition (csrc/engine.cu): c_r = the smallest
    multiple of 128 whose cost prefix w_point * s + row_ptr[s] reaches r/world
    of the total; equal shares if a range would exceed cap."""
    rp = np.asarray(row_ptr, dtype=np.int64)
    a = POINTS_PER_PARTIAL
    cap = share_cap(n, world) if cap is None else cap
    nal = (n + a - 1) // a
    total = w_point * n + float(rp[n])
    blocks = np.minimum(np.arange(nal + 1, dtype=np.int64) * a, n)
    pre = w_point * blocks.astype(np.float64) + rp[blocks].astype(np.float64)
    cuts = np.empty(world + 1, np.int64)
    cuts[0], cuts[world] = 0, n
    for r in range(1, world):
        want = total * r / world
        b = int(np.searchsorted(pre, want, side="left"))
        cuts[r] = min(b * a, n)
    if np.any(np.diff(cuts) > cap):
        eq = equal_share(n, world)
        cuts = np.minimum(np.arange(world + 1, dtype=np.int64) * eq, n)
        cuts[world] = n
    return cuts


# ---------------------------------------------------------------------------
# collectives
# ---------------------------------------------------------------------------
class NcclComm:
    """torch.distributed collectives on the current stream (NCCL on GPUs;
    gloo works for the host logic)."""

    def __init__(self, group=None):
        self.group = group

    def all_reduce_sum_(self, t):
        import torch.distributed as dist
        dist.all_reduce(t, group=self.group)

    def all_gather_(self, out, inp):
        import torch.distributed as dist
        dist.all_gather_into_tensor(out, inp, group=self.group)

    def min_host(self, value: int, device) -> int:
        import torch
        import torch.distributed as dist
        t = torch.tensor([value], dtype=torch.int64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
        return int(t.item())


class LocalGroup:
    """G ranks as threads of one process sharing one GPU.  Every collective
    is a rendezvous (threading.Barrier) plus stream-ordered device copies:
    a rank's stream waits on the events its peers recorded after producing
    their inputs, and producers wait until every consumer's copies are done
    before reusing the buffers.  Same call sequence and results as NCCL."""

    def __init__(self, world: int):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world
        self.done = [None] * world

    def comm(self, rank: int) -> "LocalComm":
        return LocalComm(self, rank)


class LocalComm:
    def __init__(self, group: LocalGroup, rank: int):
        self.g, self.rank = group, rank

    def _publish(self, item):
        import torch
        ev = torch.cuda.Event()
        ev.record()
        self.g.slots[self.rank] = (item, ev)
        self.g.barrier.wait()
        items = list(self.g.slots)
        self.g.barrier.wait()
        return items

    def _consumed(self):
        import torch
        ev = torch.cuda.Event()
        ev.record()
        self.g.done[self.rank] = ev
        self.g.barrier.wait()
        cur = torch.cuda.current_stream()
        for e in self.g.done:
            cur.wait_event(e)
        self.g.barrier.wait()

    def all_gather_(self, out, inp):
        import torch
        items = self._publish(inp)
        cur = torch.cuda.current_stream()
        m = inp.shape[0]
        for r, (t, ev) in enumerate(items):
            cur.wait_event(ev)
            out[r * m:(r + 1) * m].copy_(t)
        self._consumed()

    def all_reduce_sum_(self, t):
        import torch
        snap = t.clone()
        items = self._publish(snap)
        cur = torch.cuda.current_stream()
        t.zero_()
        for s, ev in items:  # rank order
            cur.wait_event(ev)
            t.add_(s)
        self._consumed()

    def min_host(self, value: int, device) -> int:
        items = self._publish(int(value))
        return min(v for v, _ in items)


# ---------------------------------------------------------------------------
# engine binding
# ---------------------------------------------------------------------------
class Shard:
    """Engine hooks of one rank: the Z all-reduce, the Y all-gather and the
    state gather of a relabel (optimizer.Engine._enqueue / relabel / store).
    """

    def __init__(self, rank: int, world: int, group=None, comm=None):
        self.rank, self.world, self.group = rank, world, group
        self.comm = comm if comm is not None else NcclComm(group)

    def attach(self, eng):
        import torch
        dt = dict(dtype=eng.dtype, device=eng.dev)
        self.ysend = torch.zeros((eng.cap, 2), **dt)
        self.gbuf = torch.zeros((self.world * eng.cap, 2), **dt)
        if isinstance(self.comm, NcclComm):
            # warm the communicator outside any graph capture
            self.comm.all_gather_(self.gbuf, self.ysend)
            z = torch.zeros_like(eng.zblock)
            self.comm.all_reduce_sum_(z)
            torch.cuda.synchronize()

    def reduce_z(self, eng):
        """All-reduce the per-128-slot Z partials, then their fixed-order
        sum into sched.z (the single-GPU reduction)."""
        from ._lib import call, ptr, stream
        self.comm.all_reduce_sum_(eng.zblock)
        call("bh_sum_partials", ptr(eng.zblock), eng.n_zblocks,
             ptr(eng.z_dev), stream())

    def _gather_rows(self, eng, dst):
        """dst (slot order) <- every rank's share of it."""
        from ._lib import call, ptr, stream
        self.comm.all_gather_(self.gbuf, self.ysend)
        call("bh_unpack_rows", ptr(self.gbuf), eng.cap, ptr(eng.cuts),
             self.world, eng.pt_bytes, ptr(dst), stream())

    def exchange_y(self, eng):
        """The updated Y of every share (packed by bh_step_update into
        ysend) to every rank, then the mean / bounds reduction."""
        from ._lib import call, ptr, stream
        self._gather_rows(eng, eng.y)
        call(eng.fn("bh_step_finish"), ptr(eng.y), eng.n, ptr(eng.sched),
             ptr(eng.bounds), eng.code_bits, ptr(eng.ws_upd),
             eng.ws_upd.numel(), stream())

    def gather_state(self, eng):
        """Velocity and gains of every slot (before a relabel / the store)."""
        from ._lib import call, ptr, stream
        for buf in (eng.v, eng.g):
            call("bh_pack_rows", ptr(buf), ptr(eng.part), eng.cap,
                 eng.pt_bytes, ptr(self.ysend), stream())
            self._gather_rows(eng, buf)

    def min_host(self, eng, value: int) -> int:
        return self.comm.min_host(value, eng.dev)


def run_local(world: int, make_engine, n_iter: int, timeout: float = 600.0):
    """Run `world` engines as threads on the current GPU with a LocalGroup:
    make_engine(shard) -> Engine; each thread runs n_iter eager iterations.
    Returns the engines (rank order).  Errors in any rank are re-raised."""
    import torch
    group = LocalGroup(world)
    dev = torch.cuda.current_device()
    engines = [None] * world
    errors = []

    def body(r):
        try:
            torch.cuda.set_device(dev)
            eng = make_engine(Shard(r, world, comm=group.comm(r)))
            engines[r] = eng
            eng.run(n_iter, use_graph=False)
            torch.cuda.synchronize()
        except BaseException as exc:  # pragma: no cover - surfaced below
            errors.append(exc)
            group.barrier.abort()

    threads = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout)
    if errors:
        raise errors[0]
    if any(t.is_alive() for t in threads):
        raise TimeoutError("local ranks did not finish")
    return engines
