"""Workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every library entry point on a small problem -- exact kNN, BSP,
symmetrize, the stage API (bounds, Morton, sort, build, both summarizes,
attractive, repulsive, exact repulsion, KL) and the engine (fused and
separate force passes, relabels, graph replay and eager), f32 and f64.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""

from __future__ import annotations

import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    import torch

    import paper_2212_11506_b200 as bh
    from paper_2212_11506_b200.workloads import c0

    n = int(os.environ.get("BH_SAN_N", 1024))
    iters = int(os.environ.get("BH_SAN_ITERS", 24))
    x = c0()[:n]
    for prec in ("f32", "f64"):
        xx = x.astype(np.float64) if prec == "f64" else x
        g = bh.knn_exact(xx, 30)
        pr = bh.calibrate_perplexity(g, 10.0)
        p = bh.symmetrize(pr, g, dtype=xx.dtype)
        y = bh.init_embedding(n, 0, dtype=xx.dtype).y * 1e3
        c, r = bh.compute_bounds(y)
        t = bh.summarize(bh.build_tree(bh.morton_codes(y, c, r), y))
        buf = bh.GradientBuffers.allocate(n, y.dtype)
        bh.attractive(p, y, buf)
        for theta in (0.5, 0.8):
            bh.repulsive_bh(t, y, theta, buf)
        bh.repulsive_exact(y, buf)
        bh.kl_divergence(p, y, mode="exact")
        cfg = bh.TsneConfig(n_iter=iters, exaggeration_iters=iters // 3,
                            relabel_every=7, graph_chunk=5, precision=prec)
        for fuse, graph in ((True, True), (False, False)):
            e = bh.init_embedding(n, 0, dtype=xx.dtype)
            eng = bh.Engine(p, e, cfg)
            eng.fuse = fuse
            eng.run(iters, use_graph=graph)
        if prec == "f32":
            e = bh.init_embedding(n, 0)
            eng = bh.Engine(p, e, cfg)
            eng.run(iters, bh.StepTimings())  # evented graphs
    torch.cuda.synchronize()
    print("sanitize workload ok")


if __name__ == "__main__":
    main()
