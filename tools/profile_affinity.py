"""BSP + symmetrize at C3 shape (N=1.3M, K=90) for ncu captures of k_bsp /
k_sym_*: python tools/profile_affinity.py [n].  The kNN graph is synthetic
(random ids, ascending squared distances) -- the kernels' work per row does
not depend on where the neighbours are."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2212_11506_b200 as bh  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_300_000
k = 90
rng = np.random.default_rng(0)
idx = rng.integers(0, n - 1, size=(n, k), dtype=np.int64)
idx += idx >= np.arange(n)[:, None]  # no self
sqd = np.sort(rng.gamma(4.0, 1.0, size=(n, k)).astype(np.float32), axis=1)
g = bh.NeighborGraph(indices=idx, sq_distances=sqd)
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.time()
    pr = bh.calibrate_perplexity(g, 30.0)
    torch.cuda.synchronize()
    t1 = time.time()
    p = bh.symmetrize(pr, g)
    torch.cuda.synchronize()
    t2 = time.time()
    print(f"rep {rep}: BSP {1e3 * (t1 - t0):.1f} ms, symmetrize "
          f"{1e3 * (t2 - t1):.1f} ms (host wall, incl. copies)", flush=True)
