"""Print the bench JSON line and the ncu launch list of gpurun_out/."""
import csv
import json
import sys
from collections import defaultdict

out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
for line in open(f"{out}/bench_c3.log"):
    if line.startswith("{"):
        d = json.loads(line)
        for k in ("value", "ms_per_step", "stage_ms", "kernels", "e2e", "clocks",
                  "cpu_baseline", "gpu_launches"):
            print(k, json.dumps(d.get(k))[:400])
try:
    rows = list(csv.reader(open(f"{out}/launches.csv")))
    hdr = None
    agg = defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                agg[d["Kernel Name"][:50]].append(float(d["Metric Value"].replace(",", "")))
    for k, v in agg.items():
        print(f"{k:50s} n={len(v):3d} mean_us={sum(v) / len(v) / 1000:.2f}")
except FileNotFoundError:
    pass
