"""Index locality of the CSR gathers in storage (Morton) order (GPU tool).

    python tools/attr_locality.py [--preroll 600]

For row tiles of R rows and halo W, prints the fraction of P's non-zeros
whose column lies in [tile_start - W, tile_end + W): the share of y_j
gathers a shared-memory window of the tile would serve.
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
    args = ap.parse_args()
    import numpy as np
    import torch

    import bench
    import paper_2212_11506_b200 as bh

    dev = torch.device("cuda", 0)
    prob = bench.problem(args.config, dev)
    p = bh.from_csr(prob["row_offsets"], prob["col"], prob["val"])
    cache = f"/tmp/bh_bench_cache/{args.config}_v2_y{args.preroll}.npy"
    if os.path.exists(cache):
        e = bh.embedding_from(np.load(cache))
        e.iteration = args.preroll
    else:
        e = bh.embedding_from(prob["y0"])
        bh.Engine(p, e, bh.TsneConfig()).run(args.preroll)
        np.save(cache, e.y.cpu().numpy())
    eng = bh.Engine(p, e, bh.TsneConfig())
    from paper_2212_11506_b200._lib import call, ptr, stream
    t = eng.tree
    st = stream()
    eng.load()
    eng.begin()
    call("bh_morton", ptr(eng.y), eng.n, ptr(eng.bounds), 32, 0,
         ptr(eng.codes), st)
    call("bh_sort", ptr(eng.codes), eng.n, 32, ptr(t.sorted_codes),
         ptr(t.order), ptr(eng.ws_sort), eng.ws_sort.numel(), st)
    t.build(eng.y)
    eng.relabel()
    torch.cuda.synchronize()
    rp = eng.rp.long()
    col = eng.col.long()
    n = eng.n
    counts = rp[1:n + 1] - rp[:n]
    row = torch.repeat_interleave(torch.arange(n, device=dev), counts)
    col = col[:row.numel()]
    val = eng.val[:row.numel()]
    keep = val != 0  # drop pad entries
    row, col = row[keep], col[keep]
    d = (col - row).abs().float()
    out = {"nnz": int(row.numel()),
           "median_abs_delta": float(d.median()),
           "p90_abs_delta": float(torch.quantile(d[:: max(1, d.numel() // 1000000)], 0.9))}
    for R in (256, 1024, 2048, 4096):
        for W in (1024, 2048, 4096, 8192, 16384):
            t = row // R
            lo, hi = t * R - W, t * R + R + W
            f = ((col >= lo) & (col < hi)).float().mean().item()
            out[f"R{R}_W{W}"] = round(f, 4)
    # 128-byte line sharing inside a warp-wide gather (16 points per line)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
