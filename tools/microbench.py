"""Kernel microbenchmarks on late-iteration C3 state (GPU; tuning aid).

    python tools/microbench.py [--preroll 600] [--reps 20]

Advances the C3 problem (bench.py setup cache) to a late iteration, then
times the attractive sweep and the BH traversal in isolation with CUDA
events for each value of the environment knobs given on the command line
(each run in a fresh subprocess so the library re-reads the knob).
Prints one JSON line per configuration.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def child(args):
    import numpy as np
    import torch

    import bench
    import paper_2212_11506_b200 as bh
    from paper_2212_11506_b200._lib import call, ptr, stream

    dev = torch.device("cuda", 0)
    prob = bench.problem(args.config, dev)
    p = bh.from_csr(prob["row_offsets"], prob["col"], prob["val"])
    cache = f"/tmp/bh_bench_cache/{args.config}_v2_y{args.preroll}.npy"
    cfg = bh.TsneConfig(theta=args.theta)
    if os.path.exists(cache):
        y = np.load(cache)
        e = bh.embedding_from(y)
        e.iteration = args.preroll
    else:
        e = bh.embedding_from(prob["y0"])
        eng = bh.Engine(p, e, cfg)
        eng.run(args.preroll)
        np.save(cache, e.y.cpu().numpy())
    if args.precision == "f64":  # the same state in the f64 run precision
        p = bh.from_csr(prob["row_offsets"], prob["col"],
                        prob["val"].astype(np.float64))
        e = bh.embedding_from(e.y.cpu().numpy().astype(np.float64))
        cfg = bh.TsneConfig(theta=args.theta, precision="f64")
    eng = bh.Engine(p, e, cfg)
    fn = eng.fn
    t = eng.tree
    st = stream()

    def build():
        call(fn("bh_morton"), ptr(eng.y), eng.n, ptr(eng.bounds), 32, 0,
             ptr(eng.codes), st)
        call("bh_sort", ptr(eng.codes), eng.n, 32, ptr(t.sorted_codes),
             ptr(t.order), ptr(eng.ws_sort), eng.ws_sort.numel(), st)
        t.build(eng.y)
        t.summarize()

    eng.load()
    eng.begin()
    build()
    if args.shuffle:
        # a random storage order (an input given in arbitrary order)
        g = torch.Generator(device="cpu").manual_seed(7)
        t.order.copy_(torch.randperm(eng.n, generator=g).to(torch.int32))
        eng.relabel()
    elif not args.input_order:
        eng.relabel()  # storage (Y and P) in tree order, as in the engine
    eng.begin()
    build()
    torch.cuda.synchronize()

    def timeit(fn, reps):
        fn()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        b.synchronize()
        return a.elapsed_time(b) / reps

    att = lambda: call(fn("bh_attractive"), ptr(eng.rp), ptr(eng.col), ptr(eng.val),
                       eng.n, 1, ptr(eng.y), 0, eng.n, 1.0, None, ptr(eng.attr), st)
    rep = lambda: call(fn("bh_repulsive"), t.sref(), ptr(eng.bounds), float(args.theta),
                       None, 0, eng.n, 0, ptr(eng.rep), None, None, ptr(eng.z_dev),
                       None, ptr(eng.ws_rep), eng.ws_rep.numel(), st)
    fused = lambda: call(fn("bh_forces"), t.sref(), ptr(eng.bounds), float(args.theta),
                         0, eng.n, 0, ptr(eng.rep), None, ptr(eng.z_dev),
                         ptr(eng.ws_rep), eng.ws_rep.numel(), ptr(eng.rp),
                         ptr(eng.col), ptr(eng.val), eng.n, 1, ptr(eng.y), 0,
                         eng.n, 1.0, None, ptr(eng.attr), st)

    def step_forces(mode):
        # the engine's entry point over the whole share (one GPU)
        call(fn("bh_step_forces"), t.sref(), ptr(eng.bounds),
             float(args.theta), ptr(eng.y), ptr(eng.rank_of), None,
             ptr(eng.part), eng.cap, mode, ptr(eng.rep), ptr(eng.zpart),
             ptr(eng.ws_rep), eng.ws_rep.numel(), ptr(eng.rp), ptr(eng.col),
             ptr(eng.val), 1, ptr(eng.sched), ptr(eng.attr), st)

    def sort_build():
        call("bh_sort", ptr(eng.codes), eng.n, 32, ptr(t.sorted_codes),
             ptr(t.order), ptr(eng.ws_sort), eng.ws_sort.numel(), st)
        t.build(eng.y)

    out = {"knobs": {k: v for k, v in os.environ.items() if k.startswith("BH_")},
           "iteration": args.preroll, "precision": args.precision,
           "attractive_ms": timeit(att, args.reps),
           "repulsive_ms": timeit(rep, args.reps),
           "forces_fused_ms": timeit(fused, args.reps),
           "sort_build_ms": timeit(sort_build, args.reps),

           "sort_ms": timeit(lambda: call(
               "bh_sort", ptr(eng.codes), eng.n, 32, ptr(t.sorted_codes),
               ptr(t.order), ptr(eng.ws_sort), eng.ws_sort.numel(), st),
               args.reps),
           "summarize_ms": timeit(lambda: t.summarize(), args.reps)}
    # yardstick: cuSPARSE SpMM (torch CSR @ dense) of the same relabelled P
    # with Y as the (N, 2) dense operand -- the sweep's gathers with
    # plain multiply-adds (library code, not the product path)
    try:
        pc = torch.sparse_csr_tensor(eng.rp.int(), eng.col, eng.val,
                                     size=(eng.n, eng.n))
        yy = eng.y.view(eng.n, 2).contiguous()
        out["cusparse_spmm_ms"] = timeit(lambda: torch.sparse.mm(pc, yy),
                                         args.reps)
        yx0, yx1 = yy[:, 0].contiguous(), yy[:, 1].contiguous()
        out["cusparse_2spmv_ms"] = timeit(
            lambda: (torch.mv(pc, yx0), torch.mv(pc, yx1)), args.reps)
    except Exception as exc:  # noqa: BLE001 - yardstick only
        out["cusparse_spmm_error"] = str(exc)[:200]
    out["relabel_ms"] = timeit(eng.relabel, max(2, args.reps // 4))
    if args.precision == "f32":
        out["summarize_prefix_ms"] = timeit(lambda: t.summarize_prefix(),
                                            args.reps)
        out["tree_build_prefix_ms"] = timeit(
            lambda: (t.build(eng.y), t.summarize_prefix()), args.reps)
    # the engine's force entry point on a complete tree of this state
    # (traversal of all points; fused with the sweep of rows [split, n))
    eng.begin()
    build()
    out["step_traversal_ms"] = timeit(lambda: step_forces(1), args.reps)
    out["step_fused_ms"] = timeit(lambda: step_forces(0), args.reps)
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--preroll", type=int, default=600)
    ap.add_argument("--theta", type=float, default=0.5)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--child", action="store_true")
    ap.add_argument("--input-order", action="store_true",
                    help="keep the input's storage order (a run's first 50 iterations)")
    ap.add_argument("--shuffle", action="store_true",
                    help="a random storage order (inputs in arbitrary order)")
    ap.add_argument("--precision", choices=["f32", "f64"], default="f32")
    ap.add_argument("--sweep", nargs="*", default=[],
                    help="NAME=v1,v2,... environment knobs to sweep")
    args = ap.parse_args()
    if args.child:
        return child(args)
    combos = [{}]
    for s in args.sweep:
        name, vals = s.split("=")
        combos = [dict(c, **{name: v}) for c in combos for v in vals.split(",")]
    for c in combos:
        env = dict(os.environ, **c)
        cmd = [sys.executable, __file__, "--child", "--config", args.config,
               "--preroll", str(args.preroll), "--theta", str(args.theta),
               "--reps", str(args.reps), "--precision", args.precision]
        if args.input_order:
            cmd.append("--input-order")
        if args.shuffle:
            cmd.append("--shuffle")
        subprocess.run(cmd, env=env, check=False)


if __name__ == "__main__":
    main()
