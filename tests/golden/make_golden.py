"""Generate golden vectors from the UNMODIFIED reference package.

Runs only in the build container (it imports /root/reference/pkg/src, which
does not exist on the GPU box); the outputs are committed as small .npz
fixtures next to this script and pin the oracle (tests/test_oracle.py) and
through it the CUDA path.

    python tests/golden/make_golden.py            # writes tests/golden/*.npz

Two reference modes:
  * mode 64: the reference as shipped (64-bit codes, MAX_DEPTH = 32);
  * mode 32: the reference with ``bhtsne.quadtree.MAX_DEPTH = 16`` set before
    first compilation, in a subprocess with its own NUMBA_CACHE_DIR, fed the
    64-bit codes masked to their top 32 bits -- the depth-16 oracle.
"""

from __future__ import annotations

import json
import os
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = "/root/reference/pkg/src"
REPO = os.path.dirname(os.path.dirname(HERE))


def point_sets():
    """Deterministic f32 point sets exercising the tree's edge cases."""
    sets = {}
    rng = np.random.default_rng(11)
    sets["gauss2000"] = rng.standard_normal((2000, 2)).astype(np.float32)
    # heavy tails + tight cores + exact duplicates: deep trees, depth cap binds
    rng = np.random.default_rng(12)
    core = rng.standard_normal((1500, 2)) * 1e-4
    tails = rng.standard_t(2.0, (1500, 2)) * 5.0
    dup = np.repeat(rng.standard_normal((20, 2)), 30, axis=0)
    y = np.vstack([core, tails, dup, core[:200]])  # exact repeats of the core
    sets["heavy3200"] = y[rng.permutation(y.shape[0])].astype(np.float32)
    sets["quad4"] = np.array([[-1, -1], [1, -1], [-1, 1], [1, 1]], np.float32)
    sets["dump4"] = np.array([[-1, -1], [1, -1], [-1, 1], [0.5, 0.5]],
                             np.float32)
    sets["coinc7"] = np.array([[1.0, 1.0]] * 5 + [[-1.0, -1.0]] * 2,
                              np.float32)
    sets["two"] = np.array([[0.0, 0.0], [0.0, 3.0]], np.float32)
    sets["single"] = np.array([[0.5, -0.25]], np.float32)
    return sets


TREE_FIELDS = ("level_offsets", "start", "end", "children", "is_leaf",
               "cell_center", "cell_radius", "mass", "com", "order", "ys0",
               "ys1")


def point_sets_f64():
    """float64 point sets (the reference's default run precision): values
    that are not float32-representable, plus exact duplicates."""
    sets = {}
    rng = np.random.default_rng(21)
    sets["gauss2000"] = rng.standard_normal((2000, 2))
    rng = np.random.default_rng(22)
    core = rng.standard_normal((1200, 2)) * 1e-4
    tails = rng.standard_t(2.0, (1200, 2)) * 5.0
    dup = np.repeat(rng.standard_normal((15, 2)), 20, axis=0)
    y = np.vstack([core, tails, dup])
    sets["heavy2700"] = y[rng.permutation(y.shape[0])]
    sets["coinc7"] = np.array([[1.0, 1.0]] * 5 + [[-1.0, -1.0]] * 2) + 1e-12
    sets["two"] = np.array([[0.0, 0.0], [0.1, 3.0]])
    return sets


def _tree_case(bhtsne, y, mode):
    from bhtsne import quadtree as q
    center, r_span = bhtsne.compute_bounds(y)
    mc = bhtsne.morton_codes(y, center, r_span)
    if mode == 32:
        masked = mc.codes & np.uint64(0xFFFFFFFF00000000)
        order = np.argsort(masked, kind="stable")
        mc = q.MortonCodes(codes=masked, order=order, center=mc.center,
                           r_span=mc.r_span, sorted_codes=masked[order])
    t = bhtsne.summarize(bhtsne.build_tree(mc, y))
    out = {"y": y, "center": np.array(center), "r_span": np.array(r_span),
           "codes": mc.codes, "sorted_codes": mc.sorted_codes,
           "dump": np.array(t.dump(mc.sorted_codes) if mode == 64 else "")}
    for f in TREE_FIELDS:
        out[f] = getattr(t, f)
    if y.shape[0] >= 2:
        for theta in (0.0, 0.5, 0.8):
            b = bhtsne.GradientBuffers.allocate(y.shape[0], y.dtype)
            bhtsne.repulsive_bh(t, y, theta, b)
            tag = f"bh{int(theta * 10)}"
            out[tag + "_rep0"], out[tag + "_rep1"] = b.rep0, b.rep1
            out[tag + "_zpart"], out[tag + "_z"] = b.z_partial, np.array(b.z)
        b = bhtsne.GradientBuffers.allocate(y.shape[0], y.dtype)
        bhtsne.repulsive_exact(y, b)
        out["ex_rep0"], out["ex_rep1"] = b.rep0, b.rep1
        out["ex_zpart"], out["ex_z"] = b.z_partial, np.array(b.z)
    return out


def child_trees(mode: int):
    """Subprocess body: tree fixtures in one reference mode."""
    import bhtsne
    from bhtsne import quadtree as q
    if mode == 32:
        q.MAX_DEPTH = 16
    assert q.MAX_DEPTH == (16 if mode == 32 else 32)
    for name, y in point_sets().items():
        out = _tree_case(bhtsne, y, mode)
        np.savez_compressed(os.path.join(HERE, f"tree{mode}_{name}.npz"),
                            **out)
        print(f"tree{mode}_{name}: nodes={out['start'].shape[0]}", flush=True)
    # the f64 run precision: f64 centres of mass and f64 pair terms
    for name, y in point_sets_f64().items():
        out = _tree_case(bhtsne, y, mode)
        np.savez_compressed(os.path.join(HERE, f"tree{mode}f64_{name}.npz"),
                            **out)
        print(f"tree{mode}f64_{name}: nodes={out['start'].shape[0]}",
              flush=True)


def affinity_and_forces():
    import bhtsne
    from bhtsne.affinity import SparseAffinity
    # calibrate + symmetrize + attractive on a small clustered set (f32)
    rng = np.random.default_rng(14)
    centres = rng.uniform(-5, 5, (3, 8))
    x = (centres[np.repeat(np.arange(3), 150)]
         + rng.standard_normal((450, 8))).astype(np.float32)
    g = bhtsne.knn_exact(bhtsne.InputMatrix(x), 30)
    pr = bhtsne.calibrate_perplexity(g, 10.0)
    p = bhtsne.symmetrize(pr, g, dtype=np.float32)
    y = (rng.standard_normal((450, 2)) * 3).astype(np.float32)
    buf = bhtsne.GradientBuffers.allocate(450, np.float32)
    bhtsne.attractive(p, y, buf)
    p12 = bhtsne.set_exaggeration(p, 12.0)
    buf12 = bhtsne.GradientBuffers.allocate(450, np.float32)
    bhtsne.attractive(p12, y, buf12)
    kl = bhtsne.kl_divergence(p, y)
    np.savez_compressed(
        os.path.join(HERE, "affinity450.npz"), x=x, indices=g.indices,
        sq_distances=g.sq_distances, betas=pr.betas, cond=pr.conditional,
        row_offsets=p.row_offsets, col_indices=p.col_indices, values=p.values,
        values12=p12.values, y=y, attr0=buf.attr0, attr1=buf.attr1,
        attr12_0=buf12.attr0, attr12_1=buf12.attr1, kl=np.array(kl))
    print("affinity450 nnz", p.nnz, "kl", kl)

    # gradient_step trajectory (f32 run mode), exaggerated then not
    cfg = bhtsne.TsneConfig(precision="f32", perplexity=10.0)
    e = bhtsne.init_embedding(450, seed=3, dtype=np.float32)
    traj = {"y0_init": e.y0.copy(), "y1_init": e.y1.copy()}
    pe = bhtsne.set_exaggeration(p, 12.0)
    for it in range(8):
        buffers = bhtsne.GradientBuffers.allocate(450, np.float32)
        pp = pe if it < 4 else p
        if it == 4:  # jump over the momentum switch to exercise both branches
            e.iteration = 250
        bhtsne.gradient_step(e, pp, cfg, buffers=buffers)
        traj[f"y0_{it}"], traj[f"y1_{it}"] = e.y0.copy(), e.y1.copy()
        traj[f"v0_{it}"], traj[f"g0_{it}"] = e.v0.copy(), e.g0.copy()
        traj[f"z_{it}"] = np.array(buffers.z)
    np.savez_compressed(os.path.join(HERE, "trajectory450.npz"), **traj)
    print("trajectory450 done")

    # closed forms from the reference tests re-run in f32
    y2 = np.array([[0.0, 0.0], [1.0, 0.0]], np.float32)
    p2 = SparseAffinity(n=2, row_offsets=np.array([0, 1, 2], np.int64),
                        col_indices=np.array([1, 0], np.int64),
                        values=np.array([0.5, 0.5], np.float32))
    b2 = bhtsne.GradientBuffers.allocate(2, np.float32)
    bhtsne.attractive(p2, y2, b2)
    np.savez_compressed(os.path.join(HERE, "closed_forms.npz"),
                        attr_two=b2.attr)


def affinity_f64():
    """The affinity / attractive / KL / trajectory fixtures of
    affinity_and_forces() in the reference's f64 run precision."""
    import bhtsne
    rng = np.random.default_rng(24)
    centres = rng.uniform(-5, 5, (3, 8))
    x = centres[np.repeat(np.arange(3), 150)] + rng.standard_normal((450, 8))
    g = bhtsne.knn_exact(bhtsne.InputMatrix(x), 30)
    pr = bhtsne.calibrate_perplexity(g, 10.0)
    p = bhtsne.symmetrize(pr, g, dtype=np.float64)
    y = rng.standard_normal((450, 2)) * 3
    buf = bhtsne.GradientBuffers.allocate(450, np.float64)
    bhtsne.attractive(p, y, buf)
    p12 = bhtsne.set_exaggeration(p, 12.0)
    buf12 = bhtsne.GradientBuffers.allocate(450, np.float64)
    bhtsne.attractive(p12, y, buf12)
    kl = bhtsne.kl_divergence(p, y)
    kl_bh = bhtsne.kl_divergence(p, y, mode="bh", theta=0.5)
    out = dict(x=x, indices=g.indices, sq_distances=g.sq_distances,
               betas=pr.betas, cond=pr.conditional, row_offsets=p.row_offsets,
               col_indices=p.col_indices, values=p.values, y=y,
               attr0=buf.attr0, attr1=buf.attr1, attr12_0=buf12.attr0,
               attr12_1=buf12.attr1, kl=np.array(kl), kl_bh=np.array(kl_bh))
    cfg = bhtsne.TsneConfig(precision="f64", perplexity=10.0)
    e = bhtsne.init_embedding(450, seed=3, dtype=np.float64)
    out["y0_init"], out["y1_init"] = e.y0.copy(), e.y1.copy()
    pe = bhtsne.set_exaggeration(p, 12.0)
    for it in range(8):
        buffers = bhtsne.GradientBuffers.allocate(450, np.float64)
        pp = pe if it < 4 else p
        if it == 4:  # jump over the momentum switch to exercise both branches
            e.iteration = 250
        bhtsne.gradient_step(e, pp, cfg, buffers=buffers)
        out[f"y0_{it}"], out[f"y1_{it}"] = e.y0.copy(), e.y1.copy()
        out[f"v0_{it}"], out[f"g0_{it}"] = e.v0.copy(), e.g0.copy()
        out[f"z_{it}"] = np.array(buffers.z)
    np.savez_compressed(os.path.join(HERE, "affinity450f64.npz"), **out)
    print("affinity450f64 nnz", p.nnz, "kl", kl, "kl_bh", kl_bh)


def full_run_c0():
    """C0 (BASELINE.json configs[0]) full 1000-iteration f32 run."""
    import bhtsne
    sys.path.insert(0, REPO)
    from paper_2212_11506_b200.workloads import c0
    x = c0()
    cfg = bhtsne.TsneConfig(precision="f32", seed=0, kl_every=250, threads=8)
    e, timings, kl = bhtsne.run(bhtsne.InputMatrix(x), cfg)
    g = bhtsne.knn_exact(bhtsne.InputMatrix(x), 90)
    np.savez_compressed(os.path.join(HERE, "c0_run.npz"),
                        indices=g.indices.astype(np.int16),
                        y0=e.y0, y1=e.y1, kl=np.array(kl),
                        kl_history=np.array(timings.kl_history))
    print("c0 kl", kl, timings.kl_history)


def full_run_c0_seeds():
    """C0 full f32 runs of the reference for Y0 seeds 0..7: the spread of
    the final KL over equally valid (chaotic) trajectories, beside which
    the 1% KL criterion is checked on a median (test_gpu_parity.py)."""
    import bhtsne
    sys.path.insert(0, REPO)
    from paper_2212_11506_b200.workloads import c0
    x = c0()
    kls = []
    for seed in range(8):
        cfg = bhtsne.TsneConfig(precision="f32", seed=seed, threads=8)
        _, _, kl = bhtsne.run(bhtsne.InputMatrix(x), cfg)
        kls.append(kl)
    np.savez_compressed(os.path.join(HERE, "c0_seeds.npz"),
                        seeds=np.arange(8), kl=np.array(kls))
    print("c0 seeds kl", kls)


def full_run_c1():
    """C1 (BASELINE.json configs[1], N=70k, D=50) full 1000-iteration f32
    run of the reference: its KL and periodic KL (the final-KL parity at a
    larger size; the kNN graph is recomputed from the data on the GPU)."""
    import bhtsne
    sys.path.insert(0, REPO)
    from paper_2212_11506_b200.workloads import c1
    x = c1()
    cfg = bhtsne.TsneConfig(precision="f32", seed=0, kl_every=250, threads=8)
    e, timings, kl = bhtsne.run(bhtsne.InputMatrix(x), cfg)
    np.savez_compressed(os.path.join(HERE, "c1_run.npz"), kl=np.array(kl),
                        kl_history=np.array(timings.kl_history),
                        n=np.array(x.shape[0]))
    print("c1 kl", kl, timings.kl_history)


def full_run_c2():
    """C2 (BASELINE.json configs[2], N=250k) full f32 run of the reference."""
    import bhtsne
    sys.path.insert(0, REPO)
    from paper_2212_11506_b200.workloads import c2
    x = c2()
    cfg = bhtsne.TsneConfig(precision="f32", seed=0, kl_every=250, threads=8)
    e, timings, kl = bhtsne.run(bhtsne.InputMatrix(x), cfg)
    np.savez_compressed(os.path.join(HERE, "c2_run.npz"), kl=np.array(kl),
                        kl_history=np.array(timings.kl_history),
                        n=np.array(x.shape[0]),
                        wall_s=np.array(timings.total_wall_s))
    print("c2 kl", kl, timings.kl_history, timings.total_wall_s)


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        sys.path.insert(0, REF_SRC)
        what = sys.argv[2]
        if what == "trees64":
            child_trees(64)
        elif what == "trees32":
            child_trees(32)
        elif what == "affinity":
            affinity_and_forces()
        elif what == "affinity_f64":
            affinity_f64()
        elif what == "c0":
            full_run_c0()
        elif what == "c0_seeds":
            full_run_c0_seeds()
        elif what == "c1":
            full_run_c1()
        elif what == "c2":
            full_run_c2()
        return
    jobs = sys.argv[1:] or ["trees64", "trees32", "affinity", "affinity_f64",
                            "c0"]
    for what in jobs:
        with tempfile.TemporaryDirectory() as cache:
            env = dict(os.environ, PYTHONPATH=REF_SRC, NUMBA_CACHE_DIR=cache)
            subprocess.run([sys.executable, __file__, "--child", what],
                           env=env, check=True)
    meta = {"reference": REF_SRC, "numpy": np.__version__}
    try:
        import numba
        meta["numba"] = numba.__version__
    except ImportError:
        pass
    with open(os.path.join(HERE, "MANIFEST.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


if __name__ == "__main__":
    main()
