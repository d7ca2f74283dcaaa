"""GPU timeline of the engine's fast path (tuning aid; needs a GPU).

    python tools/timeline.py [--preroll 600] [--iters 10] [--out gpurun_out/timeline.json]

Advances the C3 problem (bench.py setup, cached Y at `--preroll` like
tools/microbench.py) and records `--iters` replayed one-iteration graphs with
torch.profiler (CUPTI kernel records, also for graph-launched kernels).  Prints
per kernel: start offset within its iteration, duration, idle gap before it and
stream, then the mean per-iteration totals: busy time on the main stream, idle
gaps, the side stream's sweep.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--preroll", type=int, default=600)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--theta", type=float, default=0.5)
    ap.add_argument("--out", default=None)
    ap.add_argument("--input-order", action="store_true",
                    help="keep the input's storage order (iterations < 50 of a run)")
    args = ap.parse_args()

    import numpy as np
    import torch
    from torch.profiler import ProfilerActivity, profile

    import bench
    import paper_2212_11506_b200 as bh

    dev = torch.device("cuda", 0)
    prob = bench.problem(args.config, dev)
    p = bh.from_csr(prob["row_offsets"], prob["col"], prob["val"])
    cfg = bh.TsneConfig(theta=args.theta)
    cache = f"/tmp/bh_bench_cache/{args.config}_v2_y{args.preroll}.npy"
    if os.path.exists(cache):
        e = bh.embedding_from(np.load(cache))
        e.iteration = args.preroll
    else:
        e = bh.embedding_from(prob["y0"])
        bh.Engine(p, e, cfg).run(args.preroll)
        os.makedirs(os.path.dirname(cache), exist_ok=True)
        np.save(cache, e.y.cpu().numpy())
    eng = bh.Engine(p, e, cfg)
    # storage order = the tree order of this Y (as after a relabel), or the
    # input's own order (a run before its first relabel)
    eng.initial_relabel = not args.input_order
    eng.prepare()
    eng.run(3 if args.input_order else 20)  # warm: graphs captured
    eng.relabel_every = 0  # a relabel inside the window would skew it
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        eng.run(args.iters)
        torch.cuda.synchronize()
    evs = [ev for ev in prof.events() if ev.device_type.name == "CUDA"]
    ks = []
    for ev in evs:
        name = ev.name
        if "Memcpy" in name or "Memset" in name:
            continue
        ks.append((ev.time_range.start, ev.time_range.end, name,
                   getattr(ev, "device_index", 0)))
    ks.sort()
    if not ks:
        print("no kernel records (CUPTI unavailable?)")
        return
    # iterations: each starts with the key kernel (bh_morton / bh_hilbert)
    starts = [i for i, k in enumerate(ks) if "k_morton" in k[2]]
    rows = []
    for a, b in zip(starts, starts[1:] + [len(ks)]):
        it = ks[a:b]
        t0 = it[0][0]
        prev_end = t0
        for s, e_, name, _ in it:
            rows.append({"kernel": name.split("(")[0][:60],
                         "start_us": s - t0, "dur_us": e_ - s,
                         "gap_us": s - prev_end})
            prev_end = max(prev_end, e_)
    per_iter = [ks[b][0] - ks[a][0] for a, b in zip(starts, starts[1:])]
    # aggregate by kernel name over iterations
    agg = {}
    for r in rows:
        a = agg.setdefault(r["kernel"], [0, 0.0, 0.0, 0.0])
        a[0] += 1
        a[1] += r["dur_us"]
        a[2] += r["gap_us"]
        a[3] += r["start_us"]
    nit = max(1, len(starts))
    print(f"iterations {len(starts)}, mean iteration {np.mean(per_iter):.1f} us "
          f"(min {np.min(per_iter):.1f}, max {np.max(per_iter):.1f})")
    print(f"{'kernel':60s} {'n/it':>5s} {'start':>8s} {'dur':>8s} {'gap':>7s}")
    tot_d = tot_g = 0.0
    for name, (c, d, g, s) in sorted(agg.items(), key=lambda kv: kv[1][3] / kv[1][0]):
        print(f"{name:60s} {c / nit:5.1f} {s / c:8.1f} {d / nit:8.1f} {g / nit:7.1f}")
        tot_d += d / nit
        tot_g += g / nit
    print(f"sum of kernel time / it {tot_d:.1f} us, sum of gaps / it {tot_g:.1f} us")
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"per_iter_us": per_iter, "kernels": rows[: 80]}, f, indent=1)


if __name__ == "__main__":
    main()
