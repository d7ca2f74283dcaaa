"""C3 (BASELINE.json configs[3], N=1.3M, D=50) reference fixtures.

Run here, in the dev container (the reference is importable only here):

    python tests/golden/make_c3.py knn   # exact kNN graph -> /tmp/c3/knn.npz
    python tests/golden/make_c3.py run   # unmodified reference run() -> c3_run.npz

knn: the reference's knn_exact (knn.py:36-59) would take ~5 h on 8 cores at
N=1.3M, so the graph is computed with the same semantics faster: an f32 GEMM
filter keeps the k+M best approximate candidates per row, the candidates'
squared distances are then recomputed exactly as the reference does (f64
differences summed over the columns in order) and ranked by (distance, id)
-- the reference's strict-less insertion keeps the lower id on ties.  A row
is accepted only when the k-th exact distance lies strictly below the
smallest distance any non-candidate can have (the (k+M)-th approximate
distance minus a rigorous f32 error bound); other rows are recomputed by
brute force in f64.  The result therefore equals knn_exact bitwise.

run: the reference's own run() (optimizer.py:289-332) on the f32 data, with
knn_exact patched to return that graph (SURVEY.md 8(c) iv: verified bitwise
identical to an unpatched run on C0) and gradient_step wrapped to snapshot Y
at the start of iterations 250, 500 and 999 (the wrapper calls the
reference's gradient_step unchanged).  Saves the final exact KL, the
periodic BH KL every 250 iterations, the Y snapshots and a SHA-256 of the
kNN graph (which the GPU tests compare with the GPU kNN).
"""

from __future__ import annotations

import hashlib
import os
import sys
import tempfile
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
REF_SRC = "/root/reference/pkg/src"
WORK = "/tmp/c3"
K = 90
SNAP = (250, 500, 999)


def graph_sha(idx: np.ndarray, sqd: np.ndarray) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(idx, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(sqd, dtype=np.float32).tobytes())
    return h.hexdigest()


def exact_row(x64: np.ndarray, i: int, k: int):
    """knn.py:36-59 for one row: f64 column-ordered sums, ties -> lower id."""
    diff = x64 - x64[i]
    acc = np.zeros(x64.shape[0])
    for c in range(x64.shape[1]):  # column order, as the reference
        acc += diff[:, c] * diff[:, c]
    acc[i] = np.inf
    order = np.lexsort((np.arange(acc.shape[0]), acc))[:k]
    return order, acc[order]


def knn(x: np.ndarray, k: int = K, extra: int = 40, qb: int = 4096,
        cb: int = 65536):
    import torch
    torch.set_num_threads(os.cpu_count() or 8)
    n, d = x.shape
    x64 = x.astype(np.float64)
    xc = torch.from_numpy((x64 - x64.mean(0)).astype(np.float32))
    sq = (xc.double() ** 2).sum(1).float()
    m = k + extra
    # |err(d~)| <= g * (sq_i + sq_j + 2|x_i||x_j|) <= 2 g (sq_i + sq_j),
    # g = (d + 2) * 2^-24 per f32 dot / norm (worst-case sequential bound)
    gam = (d + 2) * 2.0 ** -24
    sqmax = float(sq.max())
    out_i = np.empty((n, k), np.int64)
    out_d = np.empty((n, k), np.float32)
    nfall = 0
    t0 = time.time()
    starts = list(range(0, n, cb))
    for qs in range(0, n, qb):
        qe = min(n, qs + qb)
        q = xc[qs:qe]
        best_v = torch.full((qe - qs, m), float("inf"))
        best_i = torch.full((qe - qs, m), -1, dtype=torch.int64)
        own = qs // cb
        order = sorted(range(len(starts)), key=lambda b: abs(b - own))
        for b in order:
            cs = starts[b]
            ce = min(n, cs + cb)
            dd = sq[qs:qe, None] + sq[None, cs:ce] - 2.0 * (q @ xc[cs:ce].T)
            if cs < qe and qs < ce:  # self pairs
                r = torch.arange(max(qs, cs), min(qe, ce))
                dd[r - qs, r - cs] = float("inf")
            tau = best_v[:, -1]
            hit = torch.nonzero(dd.amin(1) < tau).flatten()
            if hit.numel() == 0:
                continue
            sub = dd[hit]
            v, i = torch.topk(sub, min(m, sub.shape[1]), dim=1, largest=False)
            cv = torch.cat([best_v[hit], v], 1)
            ci = torch.cat([best_i[hit], i + cs], 1)
            v2, j2 = torch.topk(cv, m, dim=1, largest=False)
            best_v[hit] = v2
            best_i[hit] = torch.gather(ci, 1, j2)
        bi = best_i.numpy()
        bv = best_v.numpy().astype(np.float64)
        sqn = sq[qs:qe].double().numpy()
        for r in range(qe - qs):
            i = qs + r
            cand = bi[r]
            diff = x64[cand] - x64[i]
            acc = np.zeros(m)
            for c in range(d):
                acc += diff[:, c] * diff[:, c]
            o = np.lexsort((cand, acc))
            eps = 2.0 * gam * (sqn[r] + sqmax) * 1.01
            if acc[o[k - 1]] < bv[r, m - 1] - eps:
                out_i[i] = cand[o[:k]]
                out_d[i] = acc[o[:k]].astype(np.float32)
            else:
                nfall += 1
                oi, od = exact_row(x64, i, k)
                out_i[i] = oi
                out_d[i] = od.astype(np.float32)
        if (qs // qb) % 20 == 0:
            el = time.time() - t0
            print(f"knn rows {qe}/{n} {el:.0f}s fallback rows {nfall}",
                  flush=True)
    return out_i, out_d, nfall


def cmd_knn():
    sys.path.insert(0, REPO)
    from paper_2212_11506_b200.workloads import c3
    os.makedirs(WORK, exist_ok=True)
    x = c3()
    t0 = time.time()
    idx, sqd, nfall = knn(x)
    print(f"knn done in {time.time() - t0:.0f}s, {nfall} fallback rows")
    np.savez(os.path.join(WORK, "knn.npz"), indices=idx, sq_distances=sqd,
             wall_s=np.array(time.time() - t0), fallback_rows=np.array(nfall))


def cmd_run():
    with tempfile.TemporaryDirectory() as cache:
        os.environ["NUMBA_CACHE_DIR"] = cache
        sys.path.insert(0, REF_SRC)
        import bhtsne
        import bhtsne.optimizer as opt
        sys.path.insert(0, REPO)
        from paper_2212_11506_b200.workloads import c3
        x = c3()
        with np.load(os.path.join(WORK, "knn.npz")) as z:
            idx, sqd = z["indices"], z["sq_distances"]
        graph = bhtsne.NeighborGraph(indices=idx, sq_distances=sqd)
        opt.knn_exact = lambda xm, k: graph
        snaps = {}
        inner = opt.gradient_step
        t_iter = [time.time()]

        def step(e, p, cfg, buffers=None, timings=None):
            if e.iteration in SNAP:
                snaps[e.iteration] = np.column_stack([e.y0, e.y1]).copy()
            out = inner(e, p, cfg, buffers=buffers, timings=timings)
            if e.iteration % 50 == 0:
                print(f"it {e.iteration} {time.time() - t_iter[0]:.0f}s",
                      flush=True)
            return out

        opt.gradient_step = step
        cfg = bhtsne.TsneConfig(precision="f32", seed=0, kl_every=250,
                                threads=os.cpu_count())
        t0 = time.time()
        e, timings, kl = bhtsne.run(bhtsne.InputMatrix(x), cfg)
        wall = time.time() - t0
        print("c3 kl", kl, timings.kl_history, wall, flush=True)
        np.savez_compressed(
            os.path.join(HERE, "c3_run.npz"), kl=np.array(kl),
            kl_history=np.array(timings.kl_history), n=np.array(x.shape[0]),
            wall_s=np.array(wall), knn_sha256=np.array(graph_sha(idx, sqd)),
            snap_iterations=np.array(SNAP),
            **{f"y{t}": snaps[t].astype(np.float32) for t in SNAP},
            stage_s=np.array([timings.total(s) for s in
                              ("tree", "summarize", "attractive",
                               "repulsive", "update")]))


if __name__ == "__main__":
    {"knn": cmd_knn, "run": cmd_run}[sys.argv[1]]()
