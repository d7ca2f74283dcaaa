"""Exact GPU kNN timing (tuning aid): python tools/knn_bench.py c1 c2 ..."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2212_11506_b200 import workloads  # noqa: E402
from paper_2212_11506_b200.knn import knn_exact  # noqa: E402

import numpy as np  # noqa: E402

F64 = "--f64" in sys.argv  # float64 data (the reference's default dtype)
for name in [a for a in sys.argv[1:] if not a.startswith("--")] or ["c1"]:
    x = getattr(workloads, name)()
    if F64:
        x = x.astype(np.float64)
    torch.cuda.synchronize()
    t = time.perf_counter()
    g = knn_exact(x, 90)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    n = x.shape[0]
    print(json.dumps({"config": name, "n": n, "d": x.shape[1], "k": 90, "dtype": str(x.dtype),
                      "seconds": dt, "pairs_per_s": n * (n - 1) / dt}),
          flush=True)
