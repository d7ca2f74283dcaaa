"""Does the assignment of points to traversal warps matter?  At a late C3
iteration, times the traversal (bh_step_forces mode 1) with warps of 32
consecutive points in Morton order (the engine's order) against warps in
Hilbert order (no jumps between consecutive points) and random order.
Per-point results are identical (each lane runs its own reference walk);
only the warp unions change.

    python tools/hilbert_probe.py [--preroll 600]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def hilbert_d(x, y, order=16):
    """Hilbert distance of integer coordinates (torch int64 tensors)."""
    import torch
    d = torch.zeros_like(x)
    s = 1 << (order - 1)
    x = x.clone()
    y = y.clone()
    n = 1 << order
    while s > 0:
        rx = ((x & s) > 0).to(torch.int64)
        ry = ((y & s) > 0).to(torch.int64)
        d += s * s * ((3 * rx) ^ ry)
        # rotate
        flip = ry == 0
        swap_x = torch.where(flip & (rx == 1), n - 1 - x, x)
        swap_y = torch.where(flip & (rx == 1), n - 1 - y, y)
        x2 = torch.where(flip, swap_y, swap_x)
        y2 = torch.where(flip, swap_x, swap_y)
        x, y = x2, y2
        s >>= 1
    return d


def main():
    import torch

    import bench
    import paper_2212_11506_b200 as bh
    from paper_2212_11506_b200._lib import call, ptr, stream

    ap = argparse.ArgumentParser()
    ap.add_argument("--preroll", type=int, default=600)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    prob = bench.problem("c3", torch.device("cuda", 0))
    p = bh.from_csr(prob["row_offsets"], prob["col"], prob["val"])
    e = bh.embedding_from(prob["y0"])
    eng = bh.Engine(p, e, bh.TsneConfig())
    eng.run(args.preroll)
    eng.relabel()
    eng.run(1, use_graph=False)  # a tree of the current Y in the buffers
    torch.cuda.synchronize()
    # re-run the chain of the current state so tree, rank_of and y agree
    eng.load()
    eng.begin()
    st = stream()
    t = eng.tree
    call("bh_morton", ptr(eng.y), eng.n, ptr(eng.bounds), 32, 1,
         ptr(eng.codes), st)
    call("bh_sort", ptr(eng.codes), eng.n, 32, ptr(t.sorted_codes),
         ptr(t.order), ptr(eng.ws_sort), eng.ws_sort.numel(), st)
    t.build(eng.y, st)
    t.summarize_prefix(st)
    torch.cuda.synchronize()
    n = eng.n
    b = bh.quadtree._lib.read_struct(eng.bounds, bh.quadtree._lib.BOUNDS_DTYPE)
    yd = eng.y.double()
    q0 = ((yd[:, 0] - float(b["root0"])) * float(b["scale"])).floor().to(torch.int64)
    q1 = ((yd[:, 1] - float(b["root1"])) * float(b["scale"])).floor().to(torch.int64)
    q0 = q0.clamp(0, 65535)
    q1 = q1.clamp(0, 65535)
    hil = torch.argsort(hilbert_d(q0, q1)).to(torch.int32)
    rnd = torch.randperm(n, device=eng.dev).to(torch.int32)
    morton_list = t.order.clone()

    def run(qlist):
        call("bh_step_forces", t.sref(), ptr(eng.bounds), 0.5, ptr(eng.y),
             ptr(eng.rank_of), ptr(qlist), ptr(eng.part), n, 1, ptr(eng.rep),
             ptr(eng.zpart), ptr(eng.ws_rep), eng.ws_rep.numel(), ptr(eng.rp),
             ptr(eng.col), ptr(eng.val), 1, ptr(eng.sched), ptr(eng.attr),
             stream())

    out = {}
    ref = None
    for name, ql in (("morton_none", None), ("morton_list", morton_list),
                     ("hilbert", hil), ("random", rnd)):
        run(ql)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        c = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.reps):
            run(ql)
        c.record()
        c.synchronize()
        out[name] = a.elapsed_time(c) / args.reps
        r = eng.rep.clone()
        if ref is None:
            ref = r
        out[name + "_bitwise_same"] = bool(torch.equal(r, ref))
    # union size of 16-point warps: every warp holds 16 Hilbert-consecutive
    # points twice (2N lanes), so its walk is the union of 16 points' walks;
    # half of that kernel's time estimates a half-warp traversal's
    import ctypes as C
    import numpy as np
    h = hil.cpu().numpy()
    m = (n // 16) * 16
    dup = np.concatenate([h[:m].reshape(-1, 16), h[:m].reshape(-1, 16)],
                         axis=1).reshape(-1)
    q16 = torch.from_numpy(np.ascontiguousarray(dup)).to(eng.dev)
    part2 = torch.tensor([0, q16.numel(), q16.numel(), 1], dtype=torch.int64,
                         device=eng.dev)
    fake = type(t.struct).from_buffer_copy(t.struct)
    fake.n_points = q16.numel()
    ws2 = bh.quadtree._lib.workspace(
        bh.quadtree._lib.load().bh_repulsive_workspace_bytes(q16.numel()))

    def run16():
        call("bh_step_forces", C.byref(fake), ptr(eng.bounds), 0.5, ptr(eng.y),
             ptr(eng.rank_of), ptr(q16), ptr(part2), q16.numel(), 1,
             ptr(eng.rep), ptr(eng.zpart), ptr(ws2), ws2.numel(), ptr(eng.rp),
             ptr(eng.col), ptr(eng.val), 1, ptr(eng.sched), ptr(eng.attr),
             stream())

    run16()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    c = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(args.reps):
        run16()
    c.record()
    c.synchronize()
    out["hilbert_16pt_unions_half_time"] = a.elapsed_time(c) / args.reps / 2
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
