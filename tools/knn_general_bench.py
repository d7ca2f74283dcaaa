"""Exact GPU kNN timing outside bh_knn's fast shape (tuning aid): large k
(perplexity >= 43) and wide rows (D > 64) go through bh_knn_general."""
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2212_11506_b200 import workloads  # noqa: E402
from paper_2212_11506_b200.knn import knn_exact  # noqa: E402

rng = np.random.default_rng(0)
cases = [("c1 k=90", workloads.c1(), 90), ("c1 k=150", workloads.c1(), 150),
         ("c1 k=300", workloads.c1(), 300),
         ("70k x 100 k=90", rng.standard_normal((70_000, 100)).astype(np.float32), 90),
         ("70k x 784 k=90", rng.standard_normal((70_000, 784)).astype(np.float32), 90)]
for name, x, k in cases:
    torch.cuda.synchronize()
    t = time.perf_counter()
    knn_exact(x, k)
    torch.cuda.synchronize()
    print(json.dumps({"case": name, "seconds": round(time.perf_counter() - t, 3)}), flush=True)
