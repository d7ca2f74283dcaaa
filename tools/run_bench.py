"""Full pipeline wall time on the GPU (python tools/run_bench.py c1 c2 c3):
run(x, TsneConfig()) from the raw data -- exact kNN, BSP, P, Y0, the
1000-iteration schedule and the exact KL -- with the per-stage totals."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2212_11506_b200 as bh  # noqa: E402
from paper_2212_11506_b200 import workloads  # noqa: E402

for name in sys.argv[1:] or ["c1"]:
    x = getattr(workloads, name)()
    torch.cuda.synchronize()
    t = time.perf_counter()
    e, timings, kl = bh.run(x, bh.TsneConfig(kl_every=250))
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    rep = timings.report()
    print(json.dumps({"config": name, "n": x.shape[0], "wall_s": dt, "kl": kl,
                      "kl_history": timings.kl_history,
                      "stage_total_s": {k: round(v["total_s"], 4)
                                        for k, v in rep.items() if v["calls"]}}),
          flush=True)
