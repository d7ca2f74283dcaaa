"""Distinct 128-byte lines per warp-wide y_j gather of the attractive sweep
(GPU tool; L1 wavefronts are the attractive kernel's limit).

    python tools/attr_lines.py [--preroll 600]

Compares lane -> entry mappings on the relabelled C3 CSR (storage order):
  strided4 : lane l of a 16-lane row group loads entries 4l..4l+3 (int4),
             one gather instruction per slot (the current kernel);
  sorted   : the same with each row's columns sorted ascending;
  interleaved_sorted : lane l takes entries l, l+16, ... of a sorted row.
Prints the mean distinct lines per 32-lane gather instruction.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def lines_per_instr(addr):
    """addr: (I, 32) line ids, -1 = inactive lane -> mean distinct lines."""
    import torch
    s, _ = torch.sort(addr, dim=1)
    valid = s >= 0
    new = torch.ones_like(s, dtype=torch.bool)
    new[:, 1:] = s[:, 1:] != s[:, :-1]
    cnt = (new & valid).sum(1)
    act = valid.any(1)
    return float(cnt[act].float().mean())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--preroll", type=int, default=600)
    ap.add_argument("--rows", type=int, default=262144)
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
    if os.path.exists(cache):
        e = bh.embedding_from(np.load(cache))
    else:
        e = bh.embedding_from(prob["y0"])
        bh.Engine(p, e, bh.TsneConfig()).run(args.preroll)
        np.save(cache, e.y.cpu().numpy())
    eng = bh.Engine(p, e, bh.TsneConfig())
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
    val = eng.val
    R = min(args.rows, eng.n) // 2 * 2
    out = {"rows": R}
    G = 16
    cnt = (rp[1:R + 1] - rp[:R])
    maxlen = int(cnt.max())
    width = (maxlen + 4 * G - 1) // (4 * G) * (4 * G)
    # dense (R, width) matrix of line ids, -1 past the row end / pad entries
    idx = rp[:R, None] + torch.arange(width, device=dev)[None, :]
    inrow = torch.arange(width, device=dev)[None, :] < cnt[:, None]
    idx = torch.where(inrow, idx, torch.zeros_like(idx))
    c = torch.where(inrow & (val[idx] != 0), col[idx], torch.full_like(idx, -1))
    line = torch.where(c >= 0, c // 16, c)
    big = torch.iinfo(torch.int64).max
    srt = torch.sort(torch.where(line >= 0, line, torch.full_like(line, big)),
                     dim=1)[0]
    srt = torch.where(srt == big, torch.full_like(srt, -1), srt)

    def strided4(mat):
        # (R, width) -> instructions: rows paired, chunk j, slot s:
        # lane gl of row r reads entry 64 j + 4 gl + s
        m = mat.view(R // 2, 2, width // (4 * G), G, 4)  # pair, row, j, gl, s
        m = m.permute(0, 2, 4, 1, 3).reshape(-1, 2 * G)
        return lines_per_instr(m)

    def interleaved(mat):
        # lane gl reads entries gl, gl + 16, ...
        m = mat.view(R // 2, 2, width // G, G)
        m = m.permute(0, 2, 1, 3).reshape(-1, 2 * G)
        return lines_per_instr(m)

    out["strided4"] = strided4(line)
    out["strided4_sorted"] = strided4(srt)
    out["interleaved"] = interleaved(line)
    out["interleaved_sorted"] = interleaved(srt)
    out["mean_row_len"] = float(cnt.float().mean())
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
