"""How much gather reuse a CTA-level y staging would see in the CSR sweep:
for row blocks of R consecutive storage slots (Morton order after a
relabel) at a late C3 iteration, the number of distinct columns U per
block against the block's entries (nnz / U = reuse per staged point).

    python tools/attr_dedup.py [--preroll 600]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    import torch

    import bench
    import paper_2212_11506_b200 as bh

    ap = argparse.ArgumentParser()
    ap.add_argument("--preroll", type=int, default=600)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    prob = bench.problem("c3", torch.device("cuda", 0))
    p = bh.from_csr(prob["row_offsets"], prob["col"], prob["val"])
    e = bh.embedding_from(prob["y0"])
    eng = bh.Engine(p, e, bh.TsneConfig())
    eng.run(args.preroll)
    eng.relabel()
    torch.cuda.synchronize()
    rp, col = eng.rp, eng.col
    n = eng.n
    nnz = int(rp[-1].item())
    row = torch.repeat_interleave(torch.arange(n, device=rp.device),
                                  (rp[1:] - rp[:-1]))
    out = {"n": n, "nnz_padded": nnz, "iteration": args.preroll}
    for r in (64, 128, 256, 512, 1024, 2048):
        blk = (row // r).to(torch.int64)
        key = (blk << 32) | col[:nnz].to(torch.int64)
        key = torch.unique(key)
        ub = torch.bincount((key >> 32), minlength=(n + r - 1) // r)
        nb = torch.bincount(blk, minlength=(n + r - 1) // r)
        reuse = nb.double() / ub.clamp_min(1).double()
        out[f"R{r}"] = {
            "U_mean": float(ub.double().mean()), "U_p99": float(
                torch.quantile(ub.double(), 0.99)), "U_max": int(ub.max()),
            "nnz_per_block_mean": float(nb.double().mean()),
            "reuse_mean": float(nb.sum() / ub.sum()),
            "reuse_p1": float(torch.quantile(reuse, 0.01))}
        # column span of a block (window staging alternative)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
