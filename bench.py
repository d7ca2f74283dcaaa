"""Benchmark: BH t-SNE gradient iterations/sec at N=1.3M (BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c3|c2|c1|c0|c4] [--preroll R]

Defaults (no flags): N=1, W=5, K=995 -- the timed region is the rest of the
full 1000-iteration run (about 2-3 s of GPU time plus ~1 min of setup).
--config c4 runs the per-kernel microbench of BASELINE.json configs[4].

A step is one gradient iteration (tree build, summarize, attractive,
repulsive, update) of the full N=1.3M, D=50, K=90 problem (config C3,
synthetic data: BASELINE.json configs[3]), on the device
with inputs resident in HBM.  The timed region covers iterations
[R+W, R+W+K) of the real 1000-iteration schedule (exaggeration 12 for 250,
momentum 0.5 -> 0.8).  Setup (synthetic data, kNN graph via torch/cuBLAS,
perplexity calibration via the GPU bh_bsp, symmetrisation via a torch sort)
is identical for both arms and cached in /tmp to spare the second arm.

Prints ONE JSON line on rank 0 (see README of the driver contract): value =
whole-job iterations/s, e2e = the same through the public host-buffer API,
roofline of the dominant kernel, cpu_baseline = the CPU oracle (OpenMP
restatement of the reference) on the host cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

CACHE = "/tmp/bh_bench_cache"
FALLBACK_HBM_GBS = 6650.0


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ---------------------------------------------------------------------------
# problem setup (identical for both arms)
# ---------------------------------------------------------------------------
def knn_torch(x: np.ndarray, k: int, dev):
    """kNN graph for the benchmark inputs (setup only): fp32 distances via
    cuBLAS, top-k per row; ascending, self excluded."""
    import torch
    xt = torch.from_numpy(x).to(dev)
    n = xt.shape[0]
    sq = (xt * xt).sum(1)
    idx = torch.empty((n, k), dtype=torch.int64, device=dev)
    sqd = torch.empty((n, k), dtype=torch.float32, device=dev)
    chunk = 2048
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        d = sq[s:e, None] + sq[None, :] - 2.0 * (xt[s:e] @ xt.T)
        d[torch.arange(e - s, device=dev), torch.arange(s, e, device=dev)] = float("inf")
        v, i = torch.topk(d, k, dim=1, largest=False, sorted=True)
        idx[s:e] = i
        sqd[s:e] = v.clamp_min(0.0)
    return idx.cpu().numpy(), sqd.cpu().numpy()


def symmetrize_torch(indices, cond, dev):
    """affinity.py:121-158 semantics with a device sort (setup only)."""
    import torch
    n, k = indices.shape
    idx = torch.from_numpy(indices).to(dev)
    c = torch.from_numpy(cond).to(dev).reshape(-1)
    rows = torch.arange(n, device=dev).repeat_interleave(k)
    cols = idx.reshape(-1)
    key = torch.cat([rows * n + cols, cols * n + rows])
    val = torch.cat([c, c])
    key, order = torch.sort(key, stable=True)
    val = val[order]
    first = torch.ones_like(key, dtype=torch.bool)
    first[1:] = key[1:] != key[:-1]
    seg = torch.cumsum(first.to(torch.int64), 0) - 1
    nnz = int(seg[-1].item()) + 1
    summed = torch.zeros(nnz, dtype=torch.float64, device=dev)
    summed.index_add_(0, seg, val)
    uk = key[first]
    vals = torch.clamp(summed / (2.0 * n), min=np.finfo(np.float64).eps)
    ro = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    ro[1:] = torch.cumsum(torch.bincount(uk // n, minlength=n), 0)
    return (ro.cpu().numpy(), (uk % n).to(torch.int32).cpu().numpy(),
            vals.to(torch.float32).cpu().numpy())


def problem(config: str, dev):
    """Returns dict(n, row_offsets, col (int32), val (f32), y0 (N,2))."""
    os.makedirs(CACHE, exist_ok=True)
    path = os.path.join(CACHE, f"{config}_v2.npz")
    if os.path.exists(path):
        try:
            with np.load(path) as z:
                return {k: z[k] for k in z.files}
        except Exception:
            pass
    import paper_2212_11506_b200 as bh
    from paper_2212_11506_b200 import workloads
    t0 = time.time()
    spec = workloads.CONFIGS[config]
    x = spec["gen"]()
    log(f"[setup] {config}: data {x.shape} in {time.time() - t0:.1f}s")
    t0 = time.time()
    idx, sqd = knn_torch(x, 90, dev)
    log(f"[setup] kNN (torch) {time.time() - t0:.1f}s")
    t0 = time.time()
    pr = bh.calibrate_perplexity(
        bh.NeighborGraph(indices=idx, sq_distances=sqd), 30.0)
    cond = pr.conditional.cpu().numpy()
    log(f"[setup] BSP (GPU) {time.time() - t0:.1f}s")
    t0 = time.time()
    ro, co, va = symmetrize_torch(idx, cond, dev)
    log(f"[setup] symmetrize (torch) {time.time() - t0:.1f}s nnz={co.shape[0]}")
    # Y0 from Philox(0) as the reference's init_embedding (optimizer.py:147)
    y0 = bh.init_embedding(x.shape[0], 0).y.cpu().numpy().astype(np.float32)
    out = dict(n=np.array(x.shape[0]), row_offsets=ro, col=co, val=va, y0=y0)
    try:
        np.savez(path + ".tmp.npz", **out)
        os.replace(path + ".tmp.npz", path)
    except OSError:
        pass
    return out


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,"
              "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}",
                 f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE,
                stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        reasons = sorted({names[j] for r in self.rows for j in range(4)
                          if len(r) > 5 + j and r[5 + j].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# CPU oracle (reference restatement) timing
# ---------------------------------------------------------------------------
def cpu_oracle_time(prob, y, steps, code_bits=32):
    """Full oracle gradient iterations on the host cores from state y."""
    from oracle import oracle as o
    threads = o.set_threads(0)
    n = int(prob["n"])
    s = o.State(np.ascontiguousarray(y[:, 0]), np.ascontiguousarray(y[:, 1]),
                np.zeros(n, np.float32), np.zeros(n, np.float32),
                np.ones(n, np.float32), np.ones(n, np.float32), 0)
    ro = prob["row_offsets"]
    co = prob["col"].astype(np.int64)
    va = prob["val"]
    stage = np.zeros(5)
    tot = np.zeros(5)
    t0 = time.perf_counter()
    for _ in range(steps):
        o.gradient_step(s, ro, co, va, code_bits=code_bits, stage_s=stage)
        tot += stage
    dt = time.perf_counter() - t0
    return dt, threads, dict(zip(("tree", "summarize", "attractive",
                                  "repulsive", "update"), (tot / steps).tolist()))


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


# ---------------------------------------------------------------------------
# arms
# ---------------------------------------------------------------------------
def reference_arm(args, rank, world):
    if rank != 0:
        return
    import torch
    dev = torch.device("cuda", 0) if torch.cuda.is_available() else None
    prob = problem(args.config, dev)
    n = int(prob["n"])
    y = prob["y0"]
    w = min(args.warmup, 1)
    steps = max(1, min(args.steps, args.ref_max_steps))
    if w:
        cpu_oracle_time(prob, y, w)
    dt, threads, stages = cpu_oracle_time(prob, y, steps)
    v = steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "it/s",
        "n_gpus": world, "steps": steps, "warmup": w,
        "ms_per_step": 1e3 * dt / steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": args.precision,
        "data": "synthetic", "config": config_dict(args, n, int(prob["col"].shape[0])),
        "cpu_baseline": {"value": v, "unit": "it/s", "cores": threads,
                         "kind": "port",
                         "sample": f"{steps} full gradient iteration(s) of "
                                   f"{args.config} from Y0 on {threads} threads "
                                   f"({cpu_model()}); requested steps capped "
                                   f"at {args.ref_max_steps}",
                         "stage_s": stages},
        "e2e": {"value": v, "unit": "it/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


METRIC = "BH t-SNE gradient iters/sec at N=1.3M (1/2/4/8 B200); % of HBM roofline"


def config_dict(args, n, nnz):
    return {"workload": f"{args.config}: N={n}, D=50, K=90, perplexity 30, "
                        f"theta {args.theta}, 1000-iteration schedule "
                        f"(exaggeration 12 x 250), 32-bit Morton codes",
            "n_points": n, "nnz": nnz, "theta": args.theta,
            "timed_iterations": [args.preroll + args.warmup,
                                 args.preroll + args.warmup + args.steps],
            "l2": "inputs larger than L2 (CSR P alone > 126 MB); no flush",
            "parallelism": f"dp{args.gpus} (points/rows sharded, tree replicated)",
            "stage_breakdown": f"stage_ms/kernels: iterations [{args.preroll + args.warmup + args.steps}, "
                               f"+{args.stage_iters}) with attractive and repulsive "
                               "as separate launches, then "
                               f"+{args.stage_iters} with the fused force launch "
                               "('forces') the timed region uses",
            "fused_forces": not args.no_fuse}


def ours_arm(args, rank, world):
    import torch
    import torch.distributed as dist

    import paper_2212_11506_b200 as bh
    from paper_2212_11506_b200 import _lib

    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    prob = problem(args.config, dev)
    n = int(prob["n"])
    nnz = int(prob["col"].shape[0])
    if args.precision == "f64":  # the reference's default run precision
        prob = dict(prob, val=prob["val"].astype(np.float64),
                    y0=prob["y0"].astype(np.float64))
    p = bh.from_csr(prob["row_offsets"], prob["col"], prob["val"])
    cfg = bh.TsneConfig(theta=args.theta, graph_chunk=args.chunk,
                        precision=args.precision,
                        relabel_every=args.relabel_every)
    e = bh.embedding_from(prob["y0"])
    shard = None
    if world > 1:
        from paper_2212_11506_b200.dist import Shard
        shard = Shard(rank, world)
    eng = bh.Engine(p, e, cfg, schedule=True, shard=shard)
    eng.overlap = args.overlap
    eng.fuse = not args.no_fuse
    eng.chunk_graph = args.chunk_graph
    if args.attr_split is not None:
        eng.attr_split = args.attr_split
    eng.prepare(timings=True)  # every CUDA graph captured before timing
    if args.preroll:
        eng.run(args.preroll)
    eng.run(args.warmup)
    torch.cuda.synchronize()
    # --- timed region: K iterations, CUDA events on the launching stream
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    start = torch.cuda.Event(enable_timing=True)
    stop = torch.cuda.Event(enable_timing=True)
    launches0 = eng.launches
    with ClockSampler(local) as clk:
        start.record()
        eng.run(args.steps)
        stop.record()
        stop.synchronize()
    torch.cuda.synchronize()
    ms = start.elapsed_time(stop)
    launches = eng.launches - launches0
    # --- per-stage breakdown: the next stage_iters iterations with the
    #     evented graphs and the kernels back to back (isolated durations;
    #     outside the timed region, where the CSR sweep overlaps the chain)
    timings = bh.StepTimings()
    eng.overlap = False
    eng.run(args.stage_iters, timings)
    timings_f = bh.StepTimings()
    timings_p = bh.StepTimings()
    if eng.fuse and world == 1:
        # the fused force launch on its own (all rows), evented: the kernel
        # of the roofline; then the timed region's pipeline (side-stream
        # sweep + fused launch sharing the rows), evented: "forces" is the
        # force phase from the end of summarize to the join
        eng.fuse_timed = True
        split = eng.attr_split
        eng.attr_split = 0.0
        eng.run(args.stage_iters, timings_f)
        eng.attr_split = split
        if split:
            eng.run(args.stage_iters, timings_p)
        eng.fuse_timed = False
    eng.overlap = args.overlap
    y_start = e.y.cpu().numpy() if rank == 0 else None
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    y_end = e.y.cpu().numpy() if rank == 0 else None
    if rank != 0:
        return
    value = args.steps / (ms * 1e-3)
    stage_ms = {s: 1e3 * timings.total(s) / max(1, timings.calls(s))
                for s in ("tree", "summarize", "attractive", "repulsive",
                          "update", "comm")}
    if timings_f.calls("forces"):
        stage_ms["forces"] = 1e3 * timings_f.total("forces") / timings_f.calls("forces")
    for s_, key in (("forces", "force_phase_pipelined"),
                    ("attractive", "side_sweep_span")):
        if timings_p.calls(s_):
            stage_ms[key] = 1e3 * timings_p.total(s_) / timings_p.calls(s_)

    # --- roofline: algorithmic bytes per launch / launch time
    counts = []
    for ysnap in (y_start, y_end):
        c, r = bh.compute_bounds(ysnap)
        t = bh.summarize(bh.build_tree(bh.morton_codes(ysnap, c, r), ysnap))
        cnt = bh.repulsive_counts(t, args.theta).astype(np.int64)
        counts.append(cnt.sum(axis=0))
        del t
    cnt = np.mean(counts, axis=0)
    # 16 B per node record visited (internal + leaf), 8 B per leaf point,
    # 28 B per point (y_i, order, rep out, z) -- SURVEY.md 8(d)
    # (f64 run precision: 32 B records, 16 B points, 8 B values)
    w = 2.0 if args.precision == "f64" else 1.0
    rep_bytes = 16.0 * w * (cnt[0] + cnt[1]) + 8.0 * w * cnt[2] + (
        28.0 + 16.0 * (w - 1.0)) * n
    att_bytes = (4.0 + 4.0 * w) * nnz + 4.0 * (n + 1) + 16.0 * w * n
    peaks_path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        peak = float(json.load(open(peaks_path))["hbm_gbs"])
        peak_src = "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        peak, peak_src = FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"
    kernels = {}
    for name, b in (("repulsive", rep_bytes), ("attractive", att_bytes)):
        t_ms = stage_ms[name]
        ach = b / (t_ms * 1e-3) / 1e9
        kernels[name] = {"ms": t_ms, "algorithmic_bytes": b,
                         "achieved_gbs": ach, "frac": ach / peak}
    if stage_ms.get("forces"):
        # the fused force launch (all rows + the traversal), launched on its
        # own; in the timed region a side-stream sweep launch takes rows
        # [0, split) under the tree build and the fused launch the rest
        b = rep_bytes + att_bytes
        ach = b / (stage_ms["forces"] * 1e-3) / 1e9
        kernels["forces"] = {"ms": stage_ms["forces"], "algorithmic_bytes": b,
                             "achieved_gbs": ach, "frac": ach / peak,
                             "fused": ["attractive", "repulsive"]}
        if stage_ms.get("force_phase_pipelined"):
            kernels["forces"]["timed_region_force_phase_ms"] = stage_ms[
                "force_phase_pipelined"]
    dom = max(kernels, key=lambda k: kernels[k]["ms"])
    traffic = None
    ncu_path = os.path.join(REPO, "profiles", "ncu_traffic.json")
    if os.path.exists(ncu_path):
        try:
            tr = json.load(open(ncu_path)).get(args.config, {}).get(dom)
            traffic = None if tr is None else float(tr)
        except Exception:
            traffic = None
    roof = {"bound": "hbm", "kernel": dom,
            "achieved": kernels[dom]["achieved_gbs"], "peak": peak,
            "unit": "GB/s", "frac": kernels[dom]["frac"], "traffic": traffic,
            "peak_source": peak_src,
            # the north star's nominal ~8 TB/s, for reference
            "peak_nominal": 8000.0,
            "frac_nominal": kernels[dom]["achieved_gbs"] / 8000.0,
            "visits_per_point": (cnt[0] + cnt[1]) / n,
            "leaf_points_per_point": cnt[2] / n}

    # --- e2e through the public host-buffer API (per step: pinned host
    #     embedding state -> device, one iteration, state -> pinned host)
    runs = [e2e_run(bh, prob, cfg, args) for _ in range(max(1, args.e2e_repeats))]
    vals = sorted(r["value"] for r in runs)
    e2e = dict(runs[0], value=vals[len(vals) // 2],
               repeats=[r["value"] for r in runs],
               breakdowns=[r["breakdown_s"] for r in runs],
               clocks_per_run=[r["clocks"] for r in runs],
               summary=f"median of {len(runs)} end-to-end runs")
    e2e["per_step_host_state"] = e2e_host(bh, p, cfg, y_end, args)

    # --- CPU oracle on the host cores, bounded sample from the same state
    cpu = None
    if args.cpu_steps > 0:
        dt, threads, stages = cpu_oracle_time(prob, y_end, args.cpu_steps)
        cpu = {"value": args.cpu_steps / dt, "unit": "it/s", "cores": threads,
               "kind": "port",
               "sample": f"{args.cpu_steps} full gradient iteration(s) of "
                         f"{args.config} (N={n}) from the Y at the end of the "
                         f"timed region, C/OpenMP oracle on {threads} threads "
                         f"({cpu_model()})",
               "stage_s": stages}
    line = {
        "metric": METRIC, "value": value, "unit": "it/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": args.precision, "data": "synthetic (BASELINE.json configs[3] generator, "
                                "SURVEY.md 8(d)); kNN via cuBLAS in setup",
        "config": config_dict(args, n, nnz),
        "e2e": e2e, "gpu_launches": launches,
        "roofline": roof, "kernels": kernels, "stage_ms": stage_ms,
        "clocks": clk.summary(), "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def e2e_run(bh, prob, cfg, args):
    """End to end through the public optimiser API with HOST inputs: the
    symmetric P (CSR) and Y0 in pinned host memory are uploaded, the engine
    is built (row padding, graph capture) and runs the same W+K schedule
    iterations, and the final embedding is read back -- all inside the
    host-wall-clock timed region.  it/s = K / (time * K / (W + K))."""
    import torch
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    ro, co, va = pin(prob["row_offsets"]), pin(prob["col"]), pin(prob["val"])
    y0 = pin(prob["y0"])
    iters = args.warmup + args.steps
    # release the previous run's engine before timing this one
    import gc
    gc.collect()
    torch.cuda.synchronize()
    tick = time.perf_counter
    with ClockSampler(int(os.environ.get("LOCAL_RANK", 0))) as clk:
        t0 = tick()
        p = bh.from_csr(ro, co, va)
        e = bh.embedding_from(y0)
        torch.cuda.synchronize()
        t1 = tick()
        eng = bh.Engine(p, e, cfg)
        torch.cuda.synchronize()
        t2 = tick()
        eng.run(iters)
        torch.cuda.synchronize()
        t3 = tick()
        y_out = e.y.cpu()
        torch.cuda.synchronize()
        dt = tick() - t0
    h2d = sum(int(t.numel() * t.element_size()) for t in (ro, co, va, y0))
    d2h = int(y_out.numel() * y_out.element_size())
    return {"value": iters / dt, "unit": "it/s",
            "h2d_bytes_per_step": h2d / iters, "d2h_bytes_per_step": d2h / iters,
            "api": f"Engine(from_csr(host P), embedding_from(host Y0)).run({iters}) "
                   "+ Y to host; pinned host buffers; host wall clock incl. "
                   "upload, CSR padding, CUDA-graph capture and readback",
            "steps": iters,
            "breakdown_s": {"upload": t1 - t0, "engine_init": t2 - t1,
                            "run": t3 - t2, "readback": t0 + dt - t3},
            "clocks": clk.summary()}


def e2e_host(bh, p, cfg, y_host, args):
    import torch
    n = y_host.shape[0]
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    hy, hv, hg = pin(y_host), pin(np.zeros_like(y_host)), pin(np.ones_like(y_host))
    e = bh.embedding_from(y_host)
    eng = bh.Engine(p, e, cfg, schedule=True)
    steps = max(1, min(args.steps, args.e2e_steps))

    def one():
        e.y.copy_(hy, non_blocking=True)
        e.v.copy_(hv, non_blocking=True)
        e.g.copy_(hg, non_blocking=True)
        eng.run(1)
        hy.copy_(e.y, non_blocking=True)
        hv.copy_(e.v, non_blocking=True)
        hg.copy_(e.g, non_blocking=True)

    for _ in range(2):
        one()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    bytes_state = 3 * n * 2 * 4
    return {"value": steps / dt, "unit": "it/s",
            "h2d_bytes_per_step": bytes_state, "d2h_bytes_per_step": bytes_state,
            "api": "Engine.run(1) per step on host-resident (y, v, g): pinned "
                   "H2D, one graph-free iteration incl. bounds/centering, "
                   "D2H; host wall clock", "steps": steps}


def c4_problem(dev, n=4_000_000, k=90, seed=0):
    """BASELINE.json configs[4]: 2-D points from 100 Student-t (nu=2)
    clusters; random symmetric P with k distinct neighbours != i per row,
    values U(0,1]+1e-3 row-normalised, then symmetrised (affinity.py:121).
    The random graph is drawn with torch on the device (setup); the
    symmetrisation is our bh_symmetrize."""
    import torch

    import paper_2212_11506_b200 as bh
    from paper_2212_11506_b200 import workloads
    from paper_2212_11506_b200.affinity import PerplexityResult
    y = workloads.c4_points(seed, n)
    g = torch.Generator(device=dev)
    g.manual_seed(seed + 1)
    idx = torch.empty((n, k), dtype=torch.int64, device=dev)
    chunk = 1 << 20
    rows_all = torch.arange(n, device=dev)
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        rows = rows_all[s:e, None]
        cand = torch.randint(0, n - 1, (e - s, k), generator=g, device=dev)
        cand = cand + (cand >= rows).to(torch.int64)
        for _ in range(20):  # redraw duplicated entries until rows are distinct
            srt, order = torch.sort(cand, dim=1)
            dup = torch.zeros_like(cand, dtype=torch.bool)
            dup[:, 1:] = srt[:, 1:] == srt[:, :-1]
            if not bool(dup.any()):
                break
            redraw = torch.randint(0, n - 1, srt.shape, generator=g, device=dev)
            redraw = redraw + (redraw >= rows).to(torch.int64)
            cand = torch.where(dup, redraw, srt)
        idx[s:e] = cand
    vals = 1.0 - torch.rand((n, k), generator=g, device=dev, dtype=torch.float64)
    vals = vals + 1e-3
    vals = vals / vals.sum(dim=1, keepdim=True)
    graph = bh.NeighborGraph(idx, torch.ones((n, k), device=dev))
    pr = PerplexityResult(betas=torch.ones(n, dtype=torch.float64, device=dev),
                          conditional=vals)
    p = bh.symmetrize(pr, graph)
    return y, p


def c4_arm(args, rank, world):
    """Per-kernel microbench (no optimiser): attractive CSR sweep and the BH
    traversal at theta in {0.2, 0.5, 0.8}, GB/s of algorithmic bytes vs the
    measured HBM peak; sharded over ranks like the engine."""
    import torch
    import torch.distributed as dist

    import paper_2212_11506_b200 as bh
    from paper_2212_11506_b200 import _lib
    from paper_2212_11506_b200._lib import call, ptr, stream
    from paper_2212_11506_b200.dist import ShardPlan

    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    t0 = time.time()
    y, p = c4_problem(dev)
    torch.cuda.synchronize()
    log(f"[setup] c4 N={y.shape[0]} nnz={p.nnz} in {time.time() - t0:.1f}s")
    n, nnz = y.shape[0], p.nnz
    plan = ShardPlan(n, world, rank)
    lo, hi = plan.mine
    yt = torch.from_numpy(y).to(dev)
    c, r = bh.compute_bounds(yt)
    tree = bh.summarize(bh.build_tree(bh.morton_codes(yt, c, r), yt))
    rp, col, val = p.padded()
    attr = torch.empty((n, 2), dtype=torch.float32, device=dev)
    rep = torch.empty((n, 2), dtype=torch.float32, device=dev)
    ws = _lib.workspace(_lib.load().bh_repulsive_workspace_bytes(n))
    zt = torch.zeros(1, dtype=torch.float64, device=dev)

    def timed(fn, reps):
        fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        b.synchronize()
        ms = a.elapsed_time(b) / reps
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    try:
        peak = float(json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        peak = FALLBACK_HBM_GBS
    kernels = {}
    ms = timed(lambda: call("bh_attractive", ptr(rp), ptr(col), ptr(val), n, 1,
                            ptr(yt), lo, hi, 1.0, None, ptr(attr), stream()),
               max(3, args.steps))
    b = 8.0 * nnz + 4.0 * (n + 1) + 16.0 * n
    kernels["attractive"] = {"ms": ms, "algorithmic_bytes": b,
                             "achieved_gbs": b / ms / 1e6, "frac": b / ms / 1e6 / peak}
    for theta in (0.2, 0.5, 0.8):
        fn = lambda: call("bh_repulsive", tree.arrays.sref(), ptr(tree.bounds),
                          theta, None, lo, hi, 0, ptr(rep), None, None, ptr(zt),
                          None, ptr(ws), ws.numel(), stream())
        ms = timed(fn, max(2, args.steps // 4))
        cnt = bh.repulsive_counts(tree, theta).astype(np.int64).sum(axis=0)
        b = 16.0 * (cnt[0] + cnt[1]) + 8.0 * cnt[2] + 28.0 * n
        kernels[f"repulsive_theta{theta}"] = {
            "ms": ms, "algorithmic_bytes": b, "achieved_gbs": b / ms / 1e6,
            "frac": b / ms / 1e6 / peak, "visits_per_point": (cnt[0] + cnt[1]) / n,
            "leaf_points_per_point": cnt[2] / n}
    if rank == 0:
        print(json.dumps({
            "metric": "C4 kernel microbench: per-kernel GB/s of algorithmic "
                      "bytes vs measured HBM peak", "n_gpus": world,
            "config": {"workload": "c4: N=4M 2-D Student-t(2) mixture of 100 "
                                   "clusters, random symmetric P (K=90)",
                       "n_points": n, "nnz": nnz, "code_bits": 32},
            "peak_gbs": peak, "kernels": kernels,
            "data": "synthetic (BASELINE.json configs[4])"}), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=995)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--preroll", type=int, default=0)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3",
                    choices=["c0", "c1", "c2", "c3", "c4"])
    ap.add_argument("--theta", type=float, default=0.5)
    ap.add_argument("--precision", choices=["f32", "f64"], default="f32",
                    help="run precision (f64: the reference's default dtype)")
    ap.add_argument("--chunk", type=int, default=25)
    ap.add_argument("--cpu-steps", type=int, default=2)
    ap.add_argument("--e2e-steps", type=int, default=50)
    ap.add_argument("--e2e-repeats", type=int, default=5,
                    help="end-to-end runs through the public API (median)")
    ap.add_argument("--ref-max-steps", type=int, default=3)
    ap.add_argument("--relabel-every", type=int, default=50,
                    help="Morton relabeling period of the engine (0: never)")
    ap.add_argument("--attr-split", type=float, default=None,
                    help="fraction of CSR rows swept under the tree build")
    ap.add_argument("--chunk-graph", action="store_true",
                    help="replay one graph per graph_chunk iterations (A/B)")
    ap.add_argument("--no-fuse", action="store_true",
                    help="separate attractive/repulsive launches in the "
                         "timed region (A/B of the fused force pass)")
    ap.add_argument("--overlap", action="store_true",
                    help="CSR sweep on a side stream under the chain (A/B test)")
    ap.add_argument("--stage-iters", type=int, default=50,
                    help="iterations after the timed region measured with "
                         "per-stage events (kernel breakdown / roofline)")
    args = ap.parse_args()
    if args.warmup < 3:
        log("warmup raised to 3 (timing rules)")
        args.warmup = 3
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group("nccl")
    try:
        if args.config == "c4":
            if args.impl == "reference":
                if rank == 0:
                    print(json.dumps({"impl": "reference", "unavailable":
                                      "c4 is a GPU kernel microbench; the CPU "
                                      "oracle is reported on c3"}))
            else:
                c4_arm(args, rank, world)
        elif args.impl == "reference":
            reference_arm(args, rank, world)
        else:
            ours_arm(args, rank, world)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
