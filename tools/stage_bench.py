"""Staged CSR sweep (csrc/stage.cu) against the plain sweep on late-iteration
C3 state: build time, sweep time, bitwise equality, list statistics.

    python tools/stage_bench.py [--preroll 600] [--configs 256:13312,128:6656]
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
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--configs", default="256:13312,128:6656,512:26624")
    args = ap.parse_args()

    import numpy as np
    import torch

    import bench
    import paper_2212_11506_b200 as bh
    from paper_2212_11506_b200._lib import call, ptr, stream

    dev = torch.device("cuda", 0)
    prob = bench.problem(args.config, dev)
    p = bh.from_csr(prob["row_offsets"], prob["col"], prob["val"])
    cache = f"/tmp/bh_bench_cache/{args.config}_v2_y{args.preroll}.npy"
    cfg = bh.TsneConfig()
    if os.path.exists(cache):
        e = bh.embedding_from(np.load(cache))
        e.iteration = args.preroll
    else:
        e = bh.embedding_from(prob["y0"])
        eng = bh.Engine(p, e, cfg)
        eng.run(args.preroll)
        os.makedirs(os.path.dirname(cache), exist_ok=True)
        np.save(cache, e.y.cpu().numpy())
    eng = bh.Engine(p, e, cfg)
    t = eng.tree
    st = stream()
    eng.load()
    eng.begin()
    call("bh_morton", ptr(eng.y), eng.n, ptr(eng.bounds), 32, 0,
         ptr(eng.codes), st)
    call("bh_sort", ptr(eng.codes), eng.n, 32, ptr(t.sorted_codes),
         ptr(t.order), ptr(eng.ws_sort), eng.ws_sort.numel(), st)
    eng.relabel()
    torch.cuda.synchronize()
    n = eng.n
    nnz = eng.col.numel()

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

    plain = lambda: call("bh_attractive", ptr(eng.rp), ptr(eng.col),
                         ptr(eng.val), n, 1, ptr(eng.y), 0, n, 1.0, None,
                         ptr(eng.attr), st)
    out = {"n": n, "nnz_padded": nnz, "plain_ms": timeit(plain, args.reps)}
    ref = eng.attr.clone()
    print(json.dumps(out), flush=True)
    for c in args.configs.split(","):
        R, S = (int(x) for x in c.split(":"))
        nb = (n + R - 1) // R
        ucol = torch.zeros(nb * S, dtype=torch.int32, device=dev)
        ucount = torch.zeros(nb, dtype=torch.int32, device=dev)
        slot = torch.zeros(nnz, dtype=torch.int16, device=dev)
        build = lambda: call("bh_attr_stage_build", ptr(eng.rp), ptr(eng.col),
                             n, R, S, ptr(ucol), ptr(ucount), ptr(slot), st)
        res = {"R": R, "S": S, "smem_kb": S * 8 / 1024,
               "build_ms": timeit(build, 3)}
        out2 = torch.zeros_like(eng.attr)
        staged = lambda: call("bh_attractive_staged", ptr(eng.rp),
                              ptr(eng.col), ptr(eng.val), ptr(slot),
                              ptr(ucol), ptr(ucount), R, S, ptr(eng.y), 0, n,
                              1.0, None, ptr(out2), st)
        res["staged_ms"] = timeit(staged, args.reps)
        res["bitwise_equal"] = bool(torch.equal(out2, ref))
        uc = ucount.cpu().numpy()
        res["ucount_mean"] = float(uc.mean())
        res["ucount_max"] = int(uc.max())
        res["blocks_full"] = int((uc >= S).sum())
        res["overflow_entries"] = int((slot == -1).sum().item())
        res["reuse"] = nnz / float(uc.sum())
        # a sub-range (rows not aligned to the block size)
        lo, hi = 12345, n - 54321
        out3 = torch.zeros_like(eng.attr)
        call("bh_attractive_staged", ptr(eng.rp), ptr(eng.col), ptr(eng.val),
             ptr(slot), ptr(ucol), ptr(ucount), R, S, ptr(eng.y), lo, hi, 1.0,
             None, ptr(out3), st)
        res["subrange_equal"] = bool(torch.equal(out3[lo:hi], ref[lo:hi])
                                     and not out3[:lo].any()
                                     and not out3[hi:].any())
        print(json.dumps(res), flush=True)
        del ucol, ucount, slot


if __name__ == "__main__":
    main()
