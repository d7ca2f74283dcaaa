"""Run the engine on a clustered 200k problem for a few hundred iterations
and save the final Y (A/B bitwise comparisons of kernel variants:
`BH_LIB=variant.so python tools/traj_dump.py out.npy`)."""
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main(out, n=200_000, k=30, iters=300):
    import torch

    import paper_2212_11506_b200 as bh
    rng = np.random.default_rng(11)
    c = rng.uniform(-30, 30, (40, 2))
    y0 = (c[rng.integers(0, 40, n)] + rng.standard_t(3.0, (n, 2))).astype(np.float32) * 1e-3
    rows = np.repeat(np.arange(n), k)
    cols = (rows + rng.integers(1, 3000, n * k)) % n
    key = np.unique(np.concatenate([rows * n + cols, cols * n + rows]))
    r, cc = key // n, key % n
    v = rng.uniform(0.5, 1.5, key.shape[0])
    v = (v / v.sum()).astype(np.float32)
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=rp[1:])
    p = bh.from_csr(rp, cc.astype(np.int32), v)
    for theta in (0.5, 0.8):
        e = bh.embedding_from(y0)
        eng = bh.Engine(p, e, bh.TsneConfig(n_iter=iters, exaggeration_iters=100,
                                            theta=theta))
        eng.run(iters)
        torch.cuda.synchronize()
        np.save(out.replace(".npy", f"_t{theta}.npy"), e.y.cpu().numpy())
    print("saved", out)


if __name__ == "__main__":
    main(sys.argv[1])
