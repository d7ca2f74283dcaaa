"""Per-rank cost of the sharded engine, measured on one GPU, and the 2/4/8-GPU
projection it implies (the pool gives one GPU per call, so the multi-GPU
path cannot be timed directly).

At a C3 state (iteration --at, storage in tree order) every rank r of G
builds its sharded Engine (dist.Shard with a stand-in transport: the
all-reduce and all-gather move no data between ranks) and one iteration
is timed with CUDA events from the same restored state, --reps times:
the replicated chain (keys, sort, build, summarize of all N points), the
share's list, the side sweep and the fused force launch over the share,
the Z block sums, the share's update and the exchange kernels (pack,
unpack, Z total, mean / bounds).  Per G the heaviest rank counts.  The
NCCL transfers are added from a model: all-reduce of the Z partials
(N/128 f64) and all-gather of Y (8 B per point), at --bw GB/s of NVLink 5
bus bandwidth per GPU plus --lat_us per collective.

    python tools/multigpu_projection.py [--at 600] [--reps 20]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


class StandInComm:
    """No inter-rank data movement: the all-reduce leaves this rank's Z
    partials alone and the all-gather its own share (StandInShard fills the
    other shares with their current rows first)."""

    def __init__(self, rank):
        self.rank = rank

    def all_reduce_sum_(self, t):
        pass

    def all_gather_(self, out, inp):
        m = inp.shape[0]
        out[self.rank * m:(self.rank + 1) * m].copy_(inp)

    def min_host(self, value, device):
        return value


def stand_in_shard(rank, world):
    """A Shard whose exchanges keep the other ranks' rows as they are (a
    device-side pack of every share of the destination into the gather
    buffer before the stand-in all-gather), so the state stays a real
    embedding while only this rank's share advances."""
    from paper_2212_11506_b200._lib import call, ptr, stream
    from paper_2212_11506_b200.dist import Shard

    class StandInShard(Shard):
        prefilled = False  # set once gbuf holds every share of the state

        def prefill(self, eng, src):
            for r in range(self.world):
                call("bh_pack_rows", ptr(src), ptr(eng.parts[r]), eng.cap,
                     eng.pt_bytes, ptr(self.gbuf[r * eng.cap:]), stream())
            self.prefilled = True

        def _gather_rows(self, eng, dst):
            # before the timed graph: keep every share real by packing them
            # all; the timed iteration (its state restored before each
            # replay) leaves the other shares' gathered rows as prefilled,
            # so only this rank's own work is timed
            if not self.prefilled:
                for r in range(self.world):
                    call("bh_pack_rows", ptr(dst), ptr(eng.parts[r]), eng.cap,
                         eng.pt_bytes, ptr(self.gbuf[r * eng.cap:]), stream())
            super()._gather_rows(eng, dst)

    return StandInShard(rank, world, comm=StandInComm(rank))


def time_iteration(eng, reps):
    import torch
    snap = [t.clone() for t in (eng.y, eng.v, eng.g, eng.sched, eng.bounds)]

    def restore():
        for dst, src in zip((eng.y, eng.v, eng.g, eng.sched, eng.bounds), snap):
            dst.copy_(src)

    times = []
    if eng.shard is not None:
        eng.shard.prefill(eng, eng.y)
        torch.cuda.synchronize()
    eng.graphs.clear()  # captured after the prefill
    graph = eng._graph1()  # the fast path's one-iteration graph
    with torch.cuda.stream(eng.main):
        for _ in range(reps + 2):
            restore()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            graph.replay()
            b.record()
            b.synchronize()
            times.append(a.elapsed_time(b))
        restore()
    times = sorted(times[2:])
    # one evented replay (the timed-stage graph) for the per-stage split
    eng.fuse_timed = True
    g, evs = eng._graph(1)
    with torch.cuda.stream(eng.main):
        restore()
        g.replay()
        torch.cuda.synchronize()
        stages = {name: evs[0][a].elapsed_time(evs[0][b])
                  for name, (a, b) in eng._stage_events().items()}
        stages["iteration"] = evs[0][0].elapsed_time(evs[0][6])
        restore()
    return times[len(times) // 2], stages


def main():
    import torch

    import bench
    import paper_2212_11506_b200 as bh

    ap = argparse.ArgumentParser()
    ap.add_argument("--at", type=int, default=600)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--bw", type=float, default=700.0,
                    help="NVLink 5 bus bandwidth per GPU in a collective, GB/s")
    ap.add_argument("--lat_us", type=float, default=10.0)
    ap.add_argument("--splits", default=None,
                    help="comma-separated side-sweep fractions to time per G "
                         "(default: the engine's own choice)")
    ap.add_argument("--worlds", default="1,2,4,8")
    args = ap.parse_args()
    worlds = [int(x) for x in args.worlds.split(",")]
    splits = ([float(x) for x in args.splits.split(",")] if args.splits
              else [None])
    torch.cuda.set_device(0)
    prob = bench.problem("c3", torch.device("cuda", 0))
    p = bh.from_csr(prob["row_offsets"], prob["col"], prob["val"])
    cfg = bh.TsneConfig()
    e = bh.embedding_from(prob["y0"])
    bh.Engine(p, e, cfg).run(args.at)
    torch.cuda.synchronize()
    n = p.n
    out = {"iteration": args.at, "n": n, "model": {
        "bw_gbs": args.bw, "lat_us": args.lat_us,
        "collectives": "all-reduce of N/128 f64 Z partials + all-gather of "
                       "Y (8 B/pt), ring/NVLS cost 2(G-1)/G and (G-1)/G of "
                       "the buffer at bw, plus lat_us each"}}
    base = None
    for world, split in [(w, sp) for w in worlds for sp in splits]:
        worst, per_rank, stage_rows = 0.0, [], []
        for r in range(world):
            e2 = bh.Embedding(y=e.y.clone(), v=e.v.clone(), g=e.g.clone(),
                              iteration=e.iteration)
            shard = None if world == 1 else stand_in_shard(r, world)
            eng = bh.Engine(p, e2, cfg, shard=shard)
            if split is not None:
                eng.attr_split = split
            eng.run(1)           # builds a tree of this state
            eng.relabel()        # storage = tree order, shares re-balanced
            eng.begin()          # bounds of the centred Y, no pending shift
            torch.cuda.synchronize()
            ms, stages = time_iteration(eng, args.reps)
            eng_split = eng.attr_split
            per_rank.append(ms)
            stage_rows.append({k: round(v, 4) for k, v in stages.items()})
            worst = max(worst, ms)
            del eng
            torch.cuda.empty_cache()
        comm_ms = 0.0
        if world > 1:
            ar = 8.0 * n / 128 * 2 * (world - 1) / world
            ag = 8.0 * n * (world - 1) / world
            comm_ms = ((ar + ag) / (args.bw * 1e9)) * 1e3 + 2 * args.lat_us * 1e-3
        step = worst + comm_ms
        if base is None:
            base = step
        key = f"G{world}" if split is None else f"G{world}_split{split:g}"
        out[key] = {"attr_split": eng_split, "per_rank_ms": per_rank,
                            "max_rank_ms": worst,
                            "stages_ms_rank0": stage_rows[0],
                            "comm_model_ms": comm_ms, "step_ms": step,
                            "projected_it_s": 1e3 / step,
                            "speedup_vs_1": base / step}
        print(json.dumps({key: out[key]}), flush=True)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
