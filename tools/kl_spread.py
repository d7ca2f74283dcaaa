"""Final exact KL of the C0 pipeline over several Y0 seeds (GPU).

    python tools/kl_spread.py [--seeds 8]

The BH t-SNE trajectory is chaotic: any change in f32 summation order gives
a different (equally valid) trajectory.  This prints the final KL of
run(c0, TsneConfig(seed=s)) for s in 0..seeds-1 on the reference's kNN
graph, so the run-to-run spread can be set beside the 1% KL criterion.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=8)
    args = ap.parse_args()
    import paper_2212_11506_b200 as bh
    from paper_2212_11506_b200.workloads import c0
    x = c0()
    graph = bh.knn_exact(x, 90)  # bit-exact with the reference's knn_exact
    kls = []
    for s in range(args.seeds):
        _, _, kl = bh.run(x, bh.TsneConfig(seed=s), knn=graph)
        kls.append(float(kl))
    print(json.dumps({"config": "c0", "seeds": list(range(args.seeds)),
                      "kl": kls, "median": float(np.median(kls)),
                      "std": float(np.std(kls))}))


if __name__ == "__main__":
    main()
