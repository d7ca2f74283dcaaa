"""Gradient-descent driver on the B200: device-resident, CUDA-graph loop.

Mirrors bhtsne.optimizer (reference: pkg/src/bhtsne/optimizer.py):
``TsneConfig`` (:43-83), ``Embedding`` (:86-113), ``StepTimings``
(:116-144), ``init_embedding`` (:147-158), ``gradient_step`` (:195-224),
``kl_divergence`` (:242-270) and ``run`` (:289-332), same defaults, argument
meaning and error messages.  Differences, all deliberate:

* arrays are CUDA tensors ((N, 2) y / velocity / gains);
* ``precision`` defaults to "f32" (the north-star path: float32 storage and
  pair terms, float64 accumulation); "f64" is the reference's own default
  mode -- float64 storage and float64 pair terms in the reference's
  operation order (the library's ``_f64`` kernels);
* ``run`` takes the kNN graph (``knn=``) computed once by the reference, as
  the north star specifies, or computes it with the exact GPU kNN;
* ``code_bits`` selects 32-bit Morton codes (default) or the reference's
  64-bit codes.

The hot loop (:318-325) runs as CUDA-graph replays of ``graph_chunk``
iterations: bounds -> Morton -> radix sort -> tree -> summarize ->
attractive -> repulsive -> update, with the exaggeration / momentum schedule
read from a device-side ``bh_sched_t`` and stage times taken from external
CUDA events captured in the graph (exact per-iteration StepTimings).
"""

from __future__ import annotations

import math
import os
import time
from dataclasses import astuple, dataclass, field, replace

import numpy as np
import torch

from . import _lib
from ._lib import BOUNDS_DTYPE, SCHED_DTYPE, INT64_MAX, call, ptr, stream
from .affinity import (SparseAffinity, as_graph, calibrate_perplexity,
                       set_exaggeration, symmetrize)
from .forces import GradientBuffers, repulsive_bh, repulsive_exact
from .quadtree import (DEFAULT_CODE_BITS, TreeArrays, as_points, build_tree,
                       compute_bounds, morton_codes, summarize)

STAGES = ("knn", "bsp", "tree", "summarize", "attractive", "repulsive",
          "update")
# the stages a report lists: the reference's, plus the fused force launch
REPORT_STAGES = STAGES + ("forces",)
# "forces": the fused attractive + repulsive launch (Engine.fuse_timed)
# "iteration": start of the key pass to the end of the update (and the Y
# exchange), one event pair per iteration
EXTRA_STAGES = ("comm", "relabel", "forces", "iteration")
MOMENTUM_SWITCH_ITER = 250
PRECISIONS = ("f32", "f64")


@dataclass
class TsneConfig:
    perplexity: float = 30.0
    theta: float = 0.5
    n_iter: int = 1000
    early_exaggeration: float = 12.0
    exaggeration_iters: int = 250
    learning_rate: float = 200.0
    momentum_early: float = 0.5
    momentum_late: float = 0.8
    min_gain: float = 0.01
    seed: int = 0
    precision: str = "f32"
    threads: int | None = None  # accepted for compatibility; unused on GPU
    kl_every: int = 0
    code_bits: int = DEFAULT_CODE_BITS
    graph_chunk: int = 25
    relabel_every: int = 100  # tree-order renumbering period (0: never)
    # the engine's tree order: "hilbert" keys (the same cells and leaves as
    # the reference's Morton tree, siblings along the Hilbert curve: no
    # jumps between consecutive points, 6.5% faster traversal at C3) or
    # "morton" (the reference's sibling order); the stage API is Morton
    curve: str = "hilbert"

    def validate(self) -> "TsneConfig":
        if self.perplexity <= 1:
            raise ValueError(
                f"perplexity must be > 1, got {self.perplexity}")
        if self.theta < 0:
            raise ValueError(f"theta must be >= 0, got {self.theta}")
        if self.learning_rate <= 0:
            raise ValueError(
                f"learning rate must be > 0, got {self.learning_rate}")
        if self.n_iter < 0:
            raise ValueError(f"n_iter must be >= 0, got {self.n_iter}")
        if self.n_iter < self.exaggeration_iters:
            raise ValueError(
                f"n_iter ({self.n_iter}) must cover the exaggeration phase "
                f"({self.exaggeration_iters} iterations)")
        if self.early_exaggeration <= 0:
            raise ValueError("early exaggeration must be > 0")
        if self.precision not in PRECISIONS:
            raise ValueError(
                f"unknown precision {self.precision!r}; expected one of "
                f"{list(PRECISIONS)}")
        if self.threads is not None and self.threads < 1:
            raise ValueError(f"threads must be >= 1, got {self.threads}")
        if self.code_bits not in (32, 64):
            raise ValueError(f"code_bits must be 32 or 64, got {self.code_bits}")
        if self.graph_chunk < 1:
            raise ValueError("graph_chunk must be >= 1")
        if self.relabel_every < 0:
            raise ValueError("relabel_every must be >= 0")
        if self.curve not in ("hilbert", "morton"):
            raise ValueError(f"curve must be 'hilbert' or 'morton', got "
                             f"{self.curve!r}")
        return self

    @property
    def dtype(self):
        return np.dtype(np.float64 if self.precision == "f64" else np.float32)


@dataclass
class Embedding:
    """(N, 2) points plus optimizer state, resident on the device."""

    y: torch.Tensor   # (N, 2) float32 | float64 (the run precision)
    v: torch.Tensor   # velocity
    g: torch.Tensor   # adaptive gains (start at 1)
    iteration: int = 0
    rng_seed: int = 0

    @property
    def n_points(self) -> int:
        return self.y.shape[0]

    y0 = property(lambda s: s.y[:, 0])
    y1 = property(lambda s: s.y[:, 1])
    v0 = property(lambda s: s.v[:, 0])
    v1 = property(lambda s: s.v[:, 1])
    g0 = property(lambda s: s.g[:, 0])
    g1 = property(lambda s: s.g[:, 1])

    @property
    def velocity(self) -> torch.Tensor:
        return self.v

    @property
    def gains(self) -> torch.Tensor:
        return self.g

    def numpy(self) -> np.ndarray:
        return self.y.cpu().numpy()

    def save(self, path) -> None:
        """Checkpoint the optimiser state (y, velocity, gains, iteration,
        seed) -- what a resumed run needs (the reference has
        no checkpoint; Embedding, optimizer.py:86-97, is the state)."""
        np.savez(path, y=self.y.cpu().numpy(), v=self.v.cpu().numpy(),
                 g=self.g.cpu().numpy(), iteration=np.array(self.iteration),
                 rng_seed=np.array(self.rng_seed))

    @classmethod
    def load(cls, path) -> "Embedding":
        """Restore a checkpoint; an Engine built on it continues the schedule
        at the saved iteration (exaggeration and momentum switches)."""
        with np.load(path) as z:
            e = embedding_from(z["y"], z["v"], z["g"],
                               iteration=int(z["iteration"]))
            e.rng_seed = int(z["rng_seed"])
        return e


@dataclass
class StepTimings:
    """Wall time per pipeline stage, per call and cumulative (seconds)."""

    per_call: dict = field(
        default_factory=lambda: {s: [] for s in STAGES + EXTRA_STAGES})
    total_wall_s: float = 0.0
    kl_history: list = field(default_factory=list)

    def add(self, stage: str, seconds: float) -> None:
        self.per_call[stage].append(seconds)

    def total(self, stage: str) -> float:
        return math.fsum(self.per_call[stage])

    def calls(self, stage: str) -> int:
        return len(self.per_call[stage])

    def report(self) -> dict:
        out = {}
        for stage in STAGES + EXTRA_STAGES:
            calls = self.calls(stage)
            total = self.total(stage)
            out[stage] = {"total_s": total,
                          "per_iter_mean_s": total / calls if calls else 0.0,
                          "calls": calls}
        return out


def init_embedding(n: int, seed: int, dtype=np.float32) -> Embedding:
    """Gaussian init (sd 1e-4) from numpy's Philox(seed), as the reference,
    generated on the host (bit-identical Y0) and uploaded once."""
    if n < 2:
        raise ValueError(f"need at least 2 points, got {n}")
    dt = _lib.torch_dtype(dtype)
    rng = np.random.Generator(np.random.Philox(seed))
    y = (rng.standard_normal((n, 2)) * 1e-4).astype(
        np.float64 if dt == torch.float64 else np.float32)
    dev = _lib.device()
    yt = torch.from_numpy(np.ascontiguousarray(y)).to(dev)
    return Embedding(y=yt, v=torch.zeros_like(yt), g=torch.ones_like(yt),
                     iteration=0, rng_seed=int(seed))


def embedding_from(y, v=None, g=None, iteration=0, dtype=None) -> Embedding:
    """Embedding from host/device arrays; float64 input (or dtype) keeps the
    f64 run precision, anything else is float32."""
    pts = as_points(y, dtype).clone()
    return Embedding(y=pts,
                     v=torch.zeros_like(pts) if v is None
                     else as_points(v, pts.dtype).clone(),
                     g=torch.ones_like(pts) if g is None
                     else as_points(g, pts.dtype).clone(),
                     iteration=iteration)

# ---------------------------------------------------------------------------
# Engine: every buffer of the loop preallocated in HBM; one iteration = one
# Morton pass, the radix-sort passes, 2 tree kernels, the summarize kernels,
# the force pass (the side-stream CSR sweep + one fused launch), the update,
# enqueued on the current stream and captured in CUDA graphs.  The state is
# kept in a private "storage order", renumbered to the current Morton order
# before the first iteration and every relabel_every iterations: CSR rows,
# their column gathers and the traversal's reads and writes then touch
# nearby memory.  Results are returned in point-id order.
#
# The work is the slots / CSR rows of a bh_part_t share (device-resident):
# all of [0, n) on one GPU; on G GPUs (dist.Shard) a cost-balanced
# contiguous range per rank, with the tree rebuilt redundantly from the full
# Y, the Z partials all-reduced and the updated Y all-gathered every
# iteration.
# ---------------------------------------------------------------------------
PART_ALIGN = 128  # BH_REP_POINTS_PER_PARTIAL: one Z partial per 128 slots
# cost of a point relative to one CSR entry when balancing shares: the
# traversal (0.97 ms for 1.3M points) against the sweep (0.52 ms for 187M
# entries) at C3 -> ~270 entries per point
W_POINT = 270.0


def _align(x: int, a: int = PART_ALIGN) -> int:
    return (x + a - 1) // a * a


class Engine:
    # events: 0 start | 1 tree built | 2 summarized | 3 attractive done |
    #         4 forces done | 5 Z exchanged | 6 iteration done |
    #         7 attractive start | 8 update done (before the Y exchange) |
    #         9 traversal start (separate kernels)
    N_EVENTS = 10
    STAGE_EVENTS = {"tree": (0, 1), "summarize": (1, 2), "attractive": (7, 3),
                    "repulsive": (9, 4), "update": (5, 8)}
    STAGE_EVENTS_FUSED = {"tree": (0, 1), "summarize": (1, 2),
                          "forces": (2, 4), "update": (5, 8)}
    # with the split sweep: "attractive" = the side-stream launch (concurrent
    # with the tree build), "forces" = end of summarize to the join
    STAGE_EVENTS_FUSED_SPLIT = dict(STAGE_EVENTS_FUSED, attractive=(7, 3))

    def _fused(self, timed: bool) -> bool:
        return self.fuse and (not timed or self.fuse_timed)

    def fn(self, name: str) -> str:
        """Library entry point in the run precision."""
        return name + "_f64" if self.f64 else name

    def _stage_events(self):
        if self._fused(True):
            return (self.STAGE_EVENTS_FUSED_SPLIT if self._split_on()
                    else self.STAGE_EVENTS_FUSED)
        return (self.STAGE_EVENTS if not self._split_on()
                else dict(self.STAGE_EVENTS, attractive=(7, 3)))

    def __init__(self, p: SparseAffinity, e: Embedding, cfg: TsneConfig,
                 schedule: bool = True, shard=None):
        lib = _lib.load()
        n = e.n_points
        if p.n != n:
            raise ValueError(f"matrix is over {p.n} points, embedding has {n}")
        self.n, self.cfg, self.e, self.p = n, cfg, e, p
        self.code_bits = cfg.code_bits
        self.keys = "bh_hilbert" if cfg.curve == "hilbert" else "bh_morton"
        dev = e.y.device
        self.dev = dev
        dt = _lib.torch_dtype(cfg.precision)
        if e.y.dtype != dt:
            raise ValueError(f"embedding is {e.y.dtype} but precision is "
                             f"{cfg.precision!r}")
        self.dtype = dt
        self.f64 = dt == torch.float64
        self.pt_bytes = 16 if self.f64 else 8  # one (N, 2) row
        f2 = lambda: torch.zeros((n, 2), dtype=dt, device=dev)
        i32 = lambda: torch.zeros(n, dtype=torch.int32, device=dev)
        # storage-order state (ids[s] = point id stored at slot s)
        self.y, self.v, self.g, self.tmp = f2(), f2(), f2(), f2()
        self.ids = torch.arange(n, dtype=torch.int32, device=dev)
        self.ids_tmp, self.perm_inv = i32(), i32()
        self.rank_of = i32()  # slot -> sorted position (tree build)
        rp, col, val = p.padded()
        self.csr = {"p": (rp, col, val.to(dt))}
        self.csr_key = "p"
        self.attr, self.rep = f2(), f2()
        exag_on = schedule and cfg.n_iter > 0 and cfg.exaggeration_iters > 0
        self.sched = _lib.struct_tensor(SCHED_DTYPE, dict(
            iteration=e.iteration,
            exaggeration_iters=cfg.exaggeration_iters if exag_on else 0,
            momentum_switch=MOMENTUM_SWITCH_ITER,
            exaggeration=np.float32(cfg.early_exaggeration),
            momentum_early=cfg.momentum_early,
            momentum_late=cfg.momentum_late,
            learning_rate=cfg.learning_rate, min_gain=cfg.min_gain,
            bad=INT64_MAX, z=0.0,
            exaggeration_f64=cfg.early_exaggeration,
            momentum_early_f64=cfg.momentum_early,
            momentum_late_f64=cfg.momentum_late,
            learning_rate_f64=cfg.learning_rate, min_gain_f64=cfg.min_gain))
        self.bounds = _lib.struct_tensor(BOUNDS_DTYPE)
        self.codes = torch.zeros(
            n, dtype=torch.int32 if self.code_bits == 32 else torch.int64,
            device=dev)
        self.tree = TreeArrays(n, self.code_bits, dev, dtype=dt)
        self.tree.struct.rank = self.rank_of.data_ptr()
        self.ws_sort = _lib.workspace(lib.bh_sort_workspace_bytes(n, self.code_bits))
        self.ws_rep = _lib.workspace(lib.bh_repulsive_workspace_bytes(n))
        self.ws_upd = _lib.workspace(lib.bh_update_workspace_bytes(n))
        self.ws_bnd = _lib.workspace(lib.bh_bounds_workspace_bytes(n))
        self.ws_perm = None
        self.z_dev = self.sched[48:56].view(torch.float64)  # sched.z
        self.n_zblocks = (n + PART_ALIGN - 1) // PART_ALIGN
        self.zblock = torch.zeros(self.n_zblocks, dtype=torch.float64,
                                  device=dev)
        self.zpart = torch.zeros(n, dtype=torch.float64, device=dev)
        self.ws_zsum = _lib.workspace(lib.bh_step_zsum_workspace_bytes(n))
        self.theta = float(cfg.theta)
        self.relabel_every = cfg.relabel_every if schedule else 0
        self.since_relabel = 0
        self.relabeled = False
        self.graphs = {}
        # the iteration chain runs (and is captured) on a high-priority
        # stream; the CSR sweep on a low-priority side stream fills the SMs
        # the latency-bound chain leaves idle
        lo, hi = torch.cuda.Stream.priority_range()
        self.main = torch.cuda.Stream(device=dev, priority=hi)
        self.side = torch.cuda.Stream(device=dev, priority=lo)
        # fuse: the fast path launches the fused force pass (bh_step_forces
        # mode 0); the evented (StepTimings) path keeps the two kernels apart
        # for the per-stage breakdown unless fuse_timed is set
        self.fuse = True
        self.fuse_timed = False
        # renumber the slots in the tree order of the starting Y before the
        # first iteration (else the first relabel comes after relabel_every
        # iterations and the run starts in the input's own order)
        self.initial_relabel = os.environ.get("BH_INITIAL_RELABEL", "0") == "1"
        self.launches = 0  # library kernels enqueued by run() (bench claim)
        # False once a capture failed: a sharded engine then enqueues its
        # iterations eagerly (NCCL collectives inside CUDA graphs depend on
        # the torch / NCCL build; the single-GPU path always captures)
        self.graphs_ok = True
        # True: full chunks of the fast path replay one graph_chunk-iteration
        # graph (+0.2% device time, but capturing 25-iteration graphs for the
        # three CSR buffers costs ~0.1 s per engine: off for end-to-end runs)
        self.chunk_graph = False
        self.fork_ev = torch.cuda.Event()
        self.join_ev = torch.cuda.Event()
        # the share of this GPU (bh_part_t rows of `parts`, cuts = the
        # world + 1 boundaries); one GPU: [0, n)
        self.shard = shard
        self.world = shard.world if shard is not None else 1
        self.rank = shard.rank if shard is not None else 0
        from .dist import share_cap
        self.cap = share_cap(n, self.world)
        self.qlist = (torch.zeros(self.cap, dtype=torch.int32, device=dev)
                      if shard is not None else None)
        self.ws_q = (_lib.workspace(lib.bh_step_qlist_workspace_bytes(n))
                     if shard is not None else None)
        self.cuts = torch.zeros(self.world + 1, dtype=torch.int64, device=dev)
        self.parts = torch.zeros((self.world, 4), dtype=torch.int64, device=dev)
        self.part = self.parts[self.rank]
        # fraction of the share's CSR rows swept on the (low-priority) side
        # stream under the latency-bound tree build; the rest run inside the
        # fused force launch.  Measured at C3 (it/s, round 1): 0: 487, 0.2:
        # 612, 0.25: 614, 0.3: 619, 0.35: 620, 0.4: 618, 0.45: 613, 0.55: 602;
        # final tree, full schedule / the driver's window: 0.275: 660.9 / 634,
        # 0.3: 662.6 / 637.1, 0.325: 662.8 / 637.6, 0.35: 661.2 / 636.9
        self._attr_split = 0.325
        self._partition()
        if shard is not None:
            shard.attach(self)

    # -- the share ---------------------------------------------------------
    @property
    def attr_split(self) -> float:
        return self._attr_split

    @attr_split.setter
    def attr_split(self, frac: float):
        self._attr_split = float(frac)
        self._partition()

    def _split_on(self) -> bool:
        return self._attr_split > 0.0

    def _partition(self):
        """Balanced shares of the current storage order (device-side; the
        captured graphs read them at replay)."""
        call("bh_partition", ptr(self.rp), self.n, self.world, W_POINT,
             self._attr_split, self.cap, ptr(self.cuts), ptr(self.parts),
             stream())

    def share(self) -> tuple:
        """(lo, hi) of this GPU's slots (synchronises)."""
        p = self.part.cpu().numpy()
        return int(p[0]), int(p[1])

    @property
    def rp(self):
        return self.csr[self.csr_key][0]

    @property
    def col(self):
        return self.csr[self.csr_key][1]

    @property
    def val(self):
        return self.csr[self.csr_key][2]

    # library kernels of one relabel (invert, 4 row gathers, CSR permute:
    # 3 scan kernels + last offset + fill, partition) and of one run's load /
    # bounds / centre / store (3 gathers, 1, 1, 3 scatters)
    KERNELS_PER_RELABEL = 11
    KERNELS_PER_RUN = 8

    def kernels_per_iteration(self, timed: bool = False) -> int:
        """Library kernel launches of one iteration: morton, sort histogram +
        one pass per code byte, 2 tree kernels, the summarize kernels (2 for
        the prefix summarize; else one per level below the top 7 plus one
        for levels 6..0, tree.cu), the side sweep, the force pass (1 fused
        or 2), update; + Z sum, unpack and finish when sharded."""
        forces = 1 if self._fused(timed) else 2
        depth = self.code_bits // 2
        top = min(int(os.environ.get("BH_SUM_TOP", 6)), depth)  # tree.cu
        summarize = (2 if self.prefix_summary
                     else depth - top + (1 if top >= 0 else 0))
        return (1 + 1 + self.code_bits // 8 + 2 + summarize
                + (1 if self._split_on() else 0) + forces + 1 + 1
                + (6 if self.shard is not None else 0))

    @property
    def prefix_summary(self) -> bool:
        # f32 runs summarize from the f64 prefix sums of the sorted points
        # (2 launches; internal centres of mass differ from the reference's
        # child-order sums by f64 rounding only); f64 runs keep the
        # bit-exact level-by-level summarize.  The stage API's summarize()
        # is always the bit-exact one.
        return self.dtype == torch.float32

    # -- one iteration -----------------------------------------------------
    def _enqueue(self, ev=None):
        st = stream()
        n, cb, t = self.n, self.code_bits, self.tree
        y = self.y
        rec = (lambda i: ev[i].record()) if ev is not None else (lambda i: None)
        sharded = self.shard is not None
        fused = self._fused(ev is not None)
        rec(0)
        self._nvtx("tree")
        call(self.fn(self.keys), ptr(y), n, ptr(self.bounds), cb, 1,
             ptr(self.codes), st)
        if self._split_on():
            # rows [lo, split) of the share are swept on the side stream
            # under the latency-bound tree build (they need only Y and P)
            self.fork_ev.record(torch.cuda.current_stream())
            with torch.cuda.stream(self.side):
                self.side.wait_event(self.fork_ev)
                rec(7)
                call(self.fn("bh_step_attractive"), ptr(self.rp),
                     ptr(self.col), ptr(self.val), 1, ptr(y), ptr(self.part),
                     int(math.ceil(self.cap * self._attr_split)) + 1,
                     ptr(self.sched), ptr(self.attr), stream())
                rec(3)
                self.join_ev.record(self.side)
        call("bh_sort", ptr(self.codes), n, cb, ptr(t.sorted_codes),
             ptr(t.order), ptr(self.ws_sort), self.ws_sort.numel(), st)
        t.build(y, st)
        rec(1)
        self._nvtx("summarize")
        if self.prefix_summary:
            t.summarize_prefix(st)
        else:
            t.summarize(st)
        rec(2)
        self._nvtx("forces")
        if sharded:
            # this GPU's slots in the current Morton order
            call("bh_step_qlist", ptr(t.order), n, ptr(self.part),
                 ptr(self.qlist), ptr(self.ws_q), self.ws_q.numel(), st)

        def forces(mode):
            call(self.fn("bh_step_forces"), t.sref(), ptr(self.bounds),
                 self.theta, ptr(y), ptr(self.rank_of), ptr(self.qlist),
                 ptr(self.part), self.cap, mode, ptr(self.rep),
                 ptr(self.zpart), ptr(self.ws_rep), self.ws_rep.numel(),
                 ptr(self.rp), ptr(self.col), ptr(self.val), 1,
                 ptr(self.sched), ptr(self.attr), st)

        if fused:
            # both force passes in one launch, their CTAs sharing the SMs
            # (bitwise the same results as the two kernels)
            forces(0)
        else:
            if not self._split_on():
                rec(7)
            forces(2)  # the sweep of rows [split, hi)
            if not self._split_on():
                rec(3)
            rec(9)
            forces(1)  # the traversal
        if self._split_on():
            torch.cuda.current_stream().wait_event(self.join_ev)
        # Z: per-128-slot block sums of zpart (the other GPUs' blocks stay
        # 0 for the all-reduce); one GPU folds them into sched.z at once
        self._nvtx("z")
        if sharded:
            self.zblock.zero_()
        call("bh_step_zsum", ptr(self.zpart), ptr(self.part), n, self.cap,
             ptr(self.zblock), None if sharded else ptr(self.z_dev),
             ptr(self.ws_zsum), self.ws_zsum.numel(), st)
        rec(4)
        if sharded:
            self.shard.reduce_z(self)
        rec(5)
        self._nvtx("update")
        call(self.fn("bh_step_update"), ptr(y), ptr(self.v), ptr(self.g),
             ptr(self.attr), ptr(self.rep), ptr(self.part), n,
             ptr(self.sched), ptr(self.bounds), cb, 0 if sharded else 1,
             ptr(self.shard.ysend) if sharded else None, ptr(self.ws_upd),
             self.ws_upd.numel(), st)
        rec(8)
        if sharded:
            self._nvtx("comm")
            self.shard.exchange_y(self)
        rec(6)
        self._nvtx(None)

    _nvtx_open = False

    def _nvtx(self, name):
        """NVTX range per stage (the StepTimings keys) around the enqueue of
        an iteration: visible to nsys / ncu --nvtx on eager iterations; a
        replayed graph shows as one "iteration" range (Engine._run)."""
        if self._nvtx_open:
            torch.cuda.nvtx.range_pop()
        self._nvtx_open = name is not None
        if name is not None:
            torch.cuda.nvtx.range_push(name)

    def _capture_or_eager(self, make):
        """make() -> graph; on a failed capture of a sharded engine, fall
        back to eager iterations (returns None) instead of failing the run."""
        try:
            return make()
        except Exception as exc:  # noqa: BLE001 - re-raised without a shard
            if self.shard is None:
                raise
            import sys
            print(f"[engine] CUDA graph capture with collectives failed "
                  f"({type(exc).__name__}: {exc}); running eager iterations",
                  file=sys.stderr)
            self.graphs_ok = False
            torch.cuda.synchronize()
            return None

    def _capture(self, enqueue):
        """Capture `enqueue()` on the main stream into a CUDA graph.  The
        loop allocates nothing (every buffer is preallocated), so the capture
        skips torch.cuda.graph's pre-capture gc.collect() / empty_cache(),
        which made end-to-end runs pay 0.1-0.6 s per capture."""
        g = torch.cuda.CUDAGraph()
        self.main.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(self.main):
            g.capture_begin()
            try:
                enqueue()
            finally:
                g.capture_end()
        return g

    def _events(self, k):
        return [[torch.cuda.Event(enable_timing=True, external=True)
                 for _ in range(self.N_EVENTS)] for _ in range(k)]

    def _key(self, *head):
        return head + (self.csr_key, self._fused(head[0] == "timed"),
                       self._split_on())

    def _graph(self, k):
        key = self._key("timed", k)
        if key not in self.graphs:
            evs = self._events(k)
            g = self._capture(lambda: [self._enqueue(evs[i]) for i in range(k)])
            self.graphs[key] = (g, evs)
        return self.graphs[key]

    def _graph1(self):
        """One iteration without timing events (the fast path: replayed
        back to back, the host only syncs at chunk boundaries)."""
        key = self._key("fast")
        if key not in self.graphs:
            self.graphs[key] = self._capture(lambda: self._enqueue(None))
        return self.graphs[key]

    def _graphk(self):
        """graph_chunk iterations in one graph without timing events: one
        graph launch per chunk instead of one per iteration."""
        k = self.cfg.graph_chunk
        key = self._key("fastk", k)
        if key not in self.graphs:
            self.graphs[key] = self._capture(
                lambda: [self._enqueue(None) for _ in range(k)])
        return self.graphs[key]

    def _alloc_relabel(self):
        if "A" not in self.csr:
            rp, col, val = self.csr["p"]
            for key in ("A", "B"):
                self.csr[key] = (torch.empty_like(rp), torch.empty_like(col),
                                 torch.empty_like(val))
            self.ws_perm = _lib.workspace(
                _lib.load().bh_permute_csr_workspace_bytes(self.n))

    def prepare(self, timings: bool = False):
        """Capture every graph a run can need (all CSR buffers), so that no
        capture happens inside a timed region."""
        keys = ["p"] + (["A", "B"] if self.relabel_every else [])
        if self.relabel_every:
            self._alloc_relabel()
        cur = self.csr_key
        with torch.cuda.stream(self.main):
            for key in keys:
                self.csr_key = key
                if self._capture_or_eager(self._graph1) is None:
                    break
                if self.chunk_graph:
                    self._graphk()
                if timings:
                    self._graph(self.cfg.graph_chunk)
        self.csr_key = cur
        torch.cuda.synchronize()

    # -- storage order -----------------------------------------------------
    def _rows(self, name, src, idx, dst, nbytes=None):
        call(name, ptr(src), ptr(idx), self.n, nbytes or self.pt_bytes,
             ptr(dst), stream())

    def load(self):
        """Point-id order (Embedding) -> storage order."""
        e = self.e
        for src, dst in ((e.y, self.y), (e.v, self.v), (e.g, self.g)):
            self._rows("bh_gather_rows", src, self.ids, dst)

    def store(self):
        """Storage order -> point-id order (Embedding)."""
        if self.shard is not None:
            self.shard.gather_state(self)
        e = self.e
        for src, dst in ((self.y, e.y), (self.v, e.v), (self.g, e.g)):
            self._rows("bh_scatter_rows", src, self.ids, dst)

    def relabel(self):
        """Renumber the storage slots in the last tree's Morton order and
        re-balance the shares."""
        if self.shard is not None:
            self.shard.gather_state(self)  # v, g of every slot
        st = stream()
        order = self.tree.order
        call("bh_invert_perm", ptr(order), self.n, ptr(self.perm_inv), st)
        for buf in (self.y, self.v, self.g):
            self._rows("bh_gather_rows", buf, order, self.tmp)
            buf.copy_(self.tmp)
        self._rows("bh_gather_rows", self.ids, order, self.ids_tmp, 4)
        self.ids.copy_(self.ids_tmp)
        nxt = "A" if self.csr_key != "A" else "B"
        self._alloc_relabel()
        rp, col, val = self.csr[self.csr_key]
        orp, ocol, oval = self.csr[nxt]
        call(self.fn("bh_permute_csr"), ptr(rp), ptr(col), ptr(val),
             ptr(order), ptr(self.perm_inv), self.n, ptr(orp), ptr(ocol),
             ptr(oval), ptr(self.ws_perm), self.ws_perm.numel(), st)
        self.csr_key = nxt
        self._partition()
        self.since_relabel = 0
        self.relabeled = True

    def _initial_relabel(self):
        """Morton order of the starting Y (shift 0) as the storage order."""
        st = stream()
        n, cb, t = self.n, self.code_bits, self.tree
        call(self.fn(self.keys), ptr(self.y), n, ptr(self.bounds), cb, 0,
             ptr(self.codes), st)
        call("bh_sort", ptr(self.codes), n, cb, ptr(t.sorted_codes),
             ptr(t.order), ptr(self.ws_sort), self.ws_sort.numel(), st)
        self.relabel()
        self.launches += 2 + self.code_bits // 8 + self.KERNELS_PER_RELABEL

    # -- driver --------------------------------------------------------------
    def begin(self):
        """Bounds of the current (centred) Y, shift 0."""
        call(self.fn("bh_bounds"), ptr(self.y), self.n, self.code_bits,
             ptr(self.bounds), ptr(self.ws_bnd), self.ws_bnd.numel(), stream())

    def end(self):
        """Apply the pending re-centering of the last update."""
        call(self.fn("bh_center"), ptr(self.y), self.n, ptr(self.bounds),
             stream())

    def set_iteration(self, it: int, exaggeration: float | None = None):
        """Host override of the schedule (stage API: p carries the factor)."""
        host = _lib.read_struct(self.sched, SCHED_DTYPE).copy()
        host["iteration"] = it
        if exaggeration is not None:
            host["exaggeration"] = np.float32(exaggeration)
            host["exaggeration_f64"] = float(exaggeration)
            host["exaggeration_iters"] = np.iinfo(np.int32).max
        self.sched.copy_(torch.from_numpy(
            np.array([host], SCHED_DTYPE).view(np.uint8)).to(self.dev))

    def _check(self):
        s = _lib.read_struct(self.sched, SCHED_DTYPE)
        bad = int(s["bad"])
        if self.shard is not None:
            bad = self.shard.min_host(self, bad)
        if bad != INT64_MAX:
            slot = bad & 0xFFFFFFFF
            point = int(self.ids[slot].item())
            raise ValueError(f"non-finite gradient at point {point} "
                             f"(iteration {bad >> 32})")
        if int(self.tree.status.item()) != 0:
            raise RuntimeError("quadtree node capacity exceeded")
        return s

    def run(self, n_iter: int, timings: StepTimings | None = None,
            use_graph: bool = True):
        """Advance n_iter iterations; the Embedding is centred on return.
        Work is stream-ordered after (and before) the caller's stream."""
        if n_iter <= 0:
            return
        caller = torch.cuda.current_stream()
        self.main.wait_stream(caller)
        with torch.cuda.stream(self.main):
            self._run(n_iter, timings, use_graph)
        caller.wait_stream(self.main)

    def _run(self, n_iter, timings, use_graph):
        self.launches += self.KERNELS_PER_RUN
        self.load()
        self.begin()
        if self.relabel_every and not self.relabeled and self.initial_relabel:
            self._initial_relabel()
        done = 0
        chunk = self.cfg.graph_chunk
        while done < n_iter:
            k = min(chunk, n_iter - done)
            evs = None
            g = None
            if use_graph and self.graphs_ok and timings is None:
                if self.chunk_graph and k == self.cfg.graph_chunk:
                    g = self._capture_or_eager(self._graphk)
                    if g is not None:
                        g.replay()
                else:
                    g = self._capture_or_eager(self._graph1)
                    for _ in range(k if g is not None else 0):
                        torch.cuda.nvtx.range_push("iteration")
                        g.replay()
                        torch.cuda.nvtx.range_pop()
            elif use_graph and self.graphs_ok:
                ge = self._capture_or_eager(lambda: self._graph(k))
                if ge is not None:
                    g, evs = ge
                    g.replay()
            if g is None:  # eager (use_graph=False, or no capture possible)
                evs = self._events(k) if timings is not None else None
                for i in range(k):
                    self._enqueue(evs[i] if evs else None)
            done += k
            self.launches += k * self.kernels_per_iteration(timings is not None)
            self.since_relabel += k
            # the chunk's non-finite check comes first: a bad gradient names
            # its point through the ids of the storage order it was found in
            self.main.synchronize()
            self._check()
            if timings is not None:
                for i in range(k):
                    for name, (a, b) in self._stage_events().items():
                        timings.add(name, evs[i][a].elapsed_time(evs[i][b]) * 1e-3)
                    timings.add("iteration",
                                evs[i][0].elapsed_time(evs[i][6]) * 1e-3)
                    if self.shard is not None:
                        timings.add("comm", (evs[i][4].elapsed_time(evs[i][5])
                                             + evs[i][8].elapsed_time(evs[i][6])) * 1e-3)
            relabel = (self.relabel_every and done < n_iter
                       and self.since_relabel >= self.relabel_every)
            if relabel:
                r0 = torch.cuda.Event(enable_timing=True)
                r1 = torch.cuda.Event(enable_timing=True)
                r0.record()
                torch.cuda.nvtx.range_push("relabel")
                self.relabel()
                torch.cuda.nvtx.range_pop()
                r1.record()
                self.launches += self.KERNELS_PER_RELABEL
                if timings is not None:
                    r1.synchronize()
                    timings.add("relabel", r0.elapsed_time(r1) * 1e-3)
        self.end()
        self.store()
        self.e.iteration += n_iter

    @property
    def z(self) -> float:
        return float(_lib.read_struct(self.sched, SCHED_DTYPE)["z"])

def gradient_step(e: Embedding, p: SparseAffinity, cfg: TsneConfig,
                  buffers: GradientBuffers | None = None,
                  timings: StepTimings | None = None) -> Embedding:
    """One full iteration: tree, summarize, forces, momentum update
    (optimizer.py:195-224); the exaggeration is the one ``p`` carries."""
    cfg.validate()
    eng = getattr(e, "_engine", None)
    # the engine copies theta and the schedule constants: key its cache on
    # the config's values, so an in-place change of cfg takes effect (the
    # reference reads cfg on every step)
    snap = astuple(cfg)
    if (eng is None or eng.p.base_values is not p.base_values
            or getattr(e, "_engine_cfg", None) != snap):
        # the embedding's dtype is the run precision, as in the reference
        # (optimizer.py:200, 214)
        prec = "f64" if e.y.dtype == torch.float64 else "f32"
        run_cfg = cfg if cfg.precision == prec else replace(cfg, precision=prec)
        eng = Engine(p, e, run_cfg, schedule=False)
        e._engine = eng
        e._engine_cfg = snap
    eng.set_iteration(e.iteration, exaggeration=p.exaggeration)
    eng.run(1, timings, use_graph=False)
    if buffers is not None:
        buffers.attr.copy_(eng.attr)
        buffers.rep.copy_(eng.rep)
        buffers.z_dev.copy_(eng.z_dev)
    return e


def kl_divergence(p: SparseAffinity, y, mode: str = "exact",
                  theta: float = 0.5) -> float:
    """C = sum p_ij ln(p_ij / q_ij) over the nonzeros of p
    (optimizer.py:242-270); Z exact (O(N^2) kernel) or Barnes-Hut."""
    if p.exaggeration != 1.0:
        raise ValueError(
            f"KL divergence requires exaggeration 1, got {p.exaggeration}")
    pts = as_points(y)
    n = pts.shape[0]
    if p.n != n:
        raise ValueError(f"matrix is over {p.n} points, embedding has {n}")
    if torch.float64 in (pts.dtype, p.dtype):  # mixed inputs: promote
        pts = pts.to(torch.float64)
    buffers = GradientBuffers.allocate(n, pts.dtype)
    if mode == "exact":
        repulsive_exact(pts, buffers)
    elif mode == "bh":
        center, r_span = compute_bounds(pts)
        tree = build_tree(morton_codes(pts, center, r_span), pts)
        summarize(tree)
        repulsive_bh(tree, pts, theta, buffers)
    else:
        raise ValueError(f"unknown mode {mode!r}; expected 'exact' or 'bh'")
    lib = _lib.load()
    out = torch.zeros(1, dtype=torch.float64, device=pts.device)
    ws = _lib.workspace(lib.bh_kl_workspace_bytes(n))
    vals = p.base_values.to(pts.dtype)
    call(_lib.fn("bh_kl_rows", pts.dtype), ptr(p.row_offsets),
         ptr(p.col_indices), ptr(vals), n, 0, ptr(pts), ptr(buffers.z_dev),
         ptr(out), ptr(ws), ws.numel(), stream())
    return float(out.item())


def affinities(x, cfg: TsneConfig, knn=None, timings=None):
    """kNN graph (given, or exact on the GPU) -> BSP -> symmetrised P."""
    tick = time.perf_counter
    if knn is None:
        from .knn import knn_exact
        data = np.ascontiguousarray(getattr(x, "data", x), dtype=cfg.dtype)
        n = data.shape[0]
        k = min(int(math.floor(3 * cfg.perplexity)), n - 1)
        t0 = tick()
        knn = knn_exact(data, k)
        torch.cuda.synchronize()
        if timings is not None:
            timings.add("knn", tick() - t0)
    elif timings is not None:
        timings.add("knn", 0.0)
    graph = as_graph(knn)
    t0 = tick()
    pr = calibrate_perplexity(graph, cfg.perplexity)
    p = symmetrize(pr, graph, dtype=cfg.dtype)
    torch.cuda.synchronize()
    if timings is not None:
        timings.add("bsp", tick() - t0)
    return p, graph


def run(x, cfg: TsneConfig, *, knn=None, profile: bool = False) -> tuple:
    """Full pipeline; returns (embedding, timings, final exact KL)
    (optimizer.py:289-332).  ``knn``: a NeighborGraph / (indices,
    sq_distances) computed once by the reference (north star), else the
    exact kNN is computed on the GPU.  ``profile``: time the stages with
    separate, non-overlapping kernels (attractive and repulsive apart, no
    side-stream sweep) so that the per-stage times add up; otherwise the
    fast pipeline runs and the timings carry "forces" (the fused launch,
    end of summarize to the join) and "attractive" (the side-stream sweep,
    concurrent with the tree build)."""
    cfg.validate()
    tick = time.perf_counter
    wall0 = tick()
    timings = StepTimings()
    data = getattr(x, "data", x)
    n = int(np.shape(data)[0]) if knn is None else as_graph(knn).n_points
    p, _ = affinities(x, cfg, knn=knn, timings=timings)
    e = init_embedding(n, cfg.seed, dtype=cfg.dtype)
    eng = Engine(p, e, cfg, schedule=True)
    if profile:
        eng.fuse_timed = False
        eng.attr_split = 0.0
    else:
        eng.fuse_timed = True
    kl_history = []
    done = 0
    while done < cfg.n_iter:
        step = cfg.n_iter - done
        if cfg.kl_every:
            step = min(step, cfg.kl_every - done % cfg.kl_every)
        eng.run(step, timings)
        done += step
        if cfg.kl_every and done % cfg.kl_every == 0:
            kl_history.append((done, kl_divergence(p, e.y, mode="bh",
                                                   theta=cfg.theta)))
    kl = kl_divergence(p, e.y, mode="exact")
    timings.total_wall_s = tick() - wall0
    timings.kl_history.extend(kl_history)
    return e, timings, kl
