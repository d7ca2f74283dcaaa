"""GPU parity of the f64 run precision (the reference's default dtype,
io.py:21-30) against golden vectors from the UNMODIFIED reference run in f64
(tests/golden/make_golden.py: tree{32,64}f64_*, affinity450f64).

Tolerances: tree topology, masses and f64 centres of mass bit-exact (same
f64 sums in the same order); per-point forces and Z to 1e-12 relative (the
same f64 pair terms as the reference, summed in the warp traversal's
order); kNN, conditionals and P bitwise or to 1e-12; trajectories to 1e-9.
"""

import numpy as np
import pytest

from conftest import golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

F64_CASES = ["gauss2000", "heavy2700", "coinc7", "two"]
TOPO = ("level_offsets", "start", "end", "children", "is_leaf", "cell_center",
        "cell_radius", "mass", "com", "order", "ys0", "ys1")


@pytest.fixture(scope="module")
def bh():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2212_11506_b200 as m
    return m


def gpu_tree(bh, y, code_bits):
    c, r = bh.compute_bounds(y, code_bits)
    mc = bh.morton_codes(y, c, r, code_bits)
    return (c, r), mc, bh.summarize(bh.build_tree(mc, y))


def rel_err(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("mode", [32, 64])
@pytest.mark.parametrize("case", F64_CASES)
def test_tree_f64_bit_exact_vs_reference(bh, mode, case):
    g = golden(f"tree{mode}f64_{case}")
    y = g["y"]
    assert y.dtype == np.float64
    (c, r), mc, t = gpu_tree(bh, y, mode)
    assert t.arrays.precision == 64 and t.arrays.ys.dtype == torch.float64
    assert c == tuple(g["center"]) and r == float(g["r_span"])
    ref_codes = g["codes"] if mode == 64 else g["codes"] >> np.uint64(32)
    np.testing.assert_array_equal(mc.codes_u64(), ref_codes)
    out = t.to_reference()
    for f in TOPO:
        assert out[f].dtype == g[f].dtype or f not in ("com", "ys0", "ys1"), f
        np.testing.assert_array_equal(out[f], g[f], err_msg=f)


@pytest.mark.parametrize("mode", [32, 64])
@pytest.mark.parametrize("case", F64_CASES)
@pytest.mark.parametrize("theta", [0.0, 0.5, 0.8])
def test_repulsive_f64_vs_reference(bh, mode, case, theta):
    g = golden(f"tree{mode}f64_{case}")
    y = g["y"]
    _, _, t = gpu_tree(bh, y, mode)
    buf = bh.GradientBuffers.allocate(y.shape[0], np.float64)
    bh.repulsive_bh(t, y, theta, buf)
    tag = f"bh{int(theta * 10)}"
    ref = np.column_stack([g[tag + "_rep0"], g[tag + "_rep1"]])
    got = buf.rep.cpu().numpy()
    assert got.dtype == np.float64
    norm = np.linalg.norm(ref, axis=1)
    err = np.linalg.norm(got - ref, axis=1)
    assert (err <= 1e-12 * np.maximum(norm, 1e-6 * norm.max()) + 1e-300).all()
    np.testing.assert_allclose(buf.z_partial.cpu().numpy(), g[tag + "_zpart"],
                               rtol=1e-13)
    assert buf.z == pytest.approx(float(g[tag + "_z"]), rel=1e-13)
    # the traversal visits exactly the reference's node set: at theta 0 the
    # f64 walk degenerates to the exact sum
    ex = bh.GradientBuffers.allocate(y.shape[0], np.float64)
    bh.repulsive_exact(y, ex)
    exref = np.column_stack([g["ex_rep0"], g["ex_rep1"]])
    assert rel_err(ex.rep.cpu().numpy(), exref) < 1e-13
    assert ex.z == pytest.approx(float(g["ex_z"]), rel=1e-13)


def test_affinity_pipeline_f64_vs_reference(bh):
    from paper_2212_11506_b200.knn import knn_exact
    g = golden("affinity450f64")
    kg = knn_exact(g["x"], 30)
    assert kg.sq_distances.dtype == torch.float64
    np.testing.assert_array_equal(kg.indices.cpu().numpy(), g["indices"])
    np.testing.assert_array_equal(kg.sq_distances.cpu().numpy(),
                                  g["sq_distances"])
    pr = bh.calibrate_perplexity(kg, 10.0)
    assert np.max(np.abs(pr.betas.cpu().numpy() - g["betas"])
                  / g["betas"]) <= 1e-12
    np.testing.assert_allclose(pr.conditional.cpu().numpy(), g["cond"],
                               rtol=1e-12, atol=1e-300)
    p = bh.symmetrize(pr, kg, dtype=np.float64)
    assert p.dtype == torch.float64
    ro, co, va = p.to_reference()
    np.testing.assert_array_equal(ro, g["row_offsets"])
    np.testing.assert_array_equal(co, g["col_indices"])
    np.testing.assert_allclose(va, g["values"], rtol=1e-12, atol=0)


def test_attractive_and_kl_f64_vs_reference(bh):
    g = golden("affinity450f64")
    p = bh.from_csr(g["row_offsets"], g["col_indices"], g["values"])
    assert p.dtype == torch.float64
    for fac, a0, a1 in ((1.0, "attr0", "attr1"), (12.0, "attr12_0", "attr12_1")):
        buf = bh.GradientBuffers.allocate(450, np.float64)
        bh.attractive(bh.set_exaggeration(p, fac), g["y"], buf)
        ref = np.column_stack([g[a0], g[a1]])
        assert rel_err(buf.attr.cpu().numpy(), ref) < 1e-13
    assert bh.kl_divergence(p, g["y"]) == pytest.approx(float(g["kl"]), rel=1e-12)
    assert bh.kl_divergence(p, g["y"], mode="bh", theta=0.5) == pytest.approx(
        float(g["kl_bh"]), rel=1e-12)


def test_gradient_step_trajectory_f64_vs_reference(bh):
    """Eight reference gradient_step calls in f64 (exaggerated, then across
    the momentum switch): the f64 engine follows to 1e-9."""
    g = golden("affinity450f64")
    p = bh.from_csr(g["row_offsets"], g["col_indices"], g["values"])
    pe = bh.set_exaggeration(p, 12.0)
    e = bh.embedding_from(np.column_stack([g["y0_init"], g["y1_init"]]))
    assert e.y.dtype == torch.float64
    cfg = bh.TsneConfig(perplexity=10.0, code_bits=64, precision="f64")
    for it in range(8):
        if it == 4:
            e.iteration = 250
        buf = bh.GradientBuffers.allocate(450, np.float64)
        bh.gradient_step(e, pe if it < 4 else p, cfg, buffers=buf)
        ref = np.column_stack([g[f"y0_{it}"], g[f"y1_{it}"]])
        assert rel_err(e.y.cpu().numpy(), ref) < 1e-9, it
        assert rel_err(e.v.cpu().numpy()[:, 0], g[f"v0_{it}"]) < 1e-9, it
        np.testing.assert_array_equal(e.g.cpu().numpy()[:, 0], g[f"g0_{it}"])
        assert buf.z == pytest.approx(float(g[f"z_{it}"]), rel=1e-12)


@pytest.mark.parametrize("code_bits", [32, 64])
def test_engine_f64_graph_relabel_and_f32_agreement(bh, code_bits):
    """The f64 engine (CUDA graphs, Morton relabeling, both code widths) is
    deterministic, equals the eager path, and reaches the f32 engine's
    objective (trajectories themselves diverge: t-SNE is chaotic)."""
    g = golden("affinity450f64")
    p = bh.from_csr(g["row_offsets"], g["col_indices"], g["values"])
    y0 = np.column_stack([g["y0_init"], g["y1_init"]])
    outs = []
    for use_graph in (True, True, False):
        e = bh.embedding_from(y0)
        cfg = bh.TsneConfig(n_iter=120, exaggeration_iters=40, graph_chunk=9,
                            code_bits=code_bits, precision="f64",
                            relabel_every=20)
        bh.Engine(p, e, cfg).run(120, use_graph=use_graph)
        outs.append(e.y.cpu().numpy().copy())
    np.testing.assert_array_equal(outs[0], outs[1])
    np.testing.assert_array_equal(outs[0], outs[2])
    # the f32 engine on the same problem stays close over 120 iterations
    e32 = bh.embedding_from(y0.astype(np.float32))
    p32 = bh.from_csr(g["row_offsets"], g["col_indices"],
                      g["values"].astype(np.float32))
    cfg32 = bh.TsneConfig(n_iter=120, exaggeration_iters=40,
                          code_bits=code_bits)
    bh.Engine(p32, e32, cfg32).run(120)
    kl64 = bh.kl_divergence(p, outs[0])
    kl32 = bh.kl_divergence(p32, e32.y)
    assert abs(kl64 - kl32) / kl32 < 0.05, (kl64, kl32)


def test_run_f64_end_to_end(bh):
    """run() in the f64 precision from raw data: f64 kNN, BSP, P, Y0, loop
    and exact KL; close to the f32 run's KL."""
    from paper_2212_11506_b200.workloads import c0
    x = c0()[:1024].astype(np.float64)
    cfg = bh.TsneConfig(n_iter=300, exaggeration_iters=100, precision="f64",
                        kl_every=100)
    e, timings, kl = bh.run(x, cfg)
    assert e.y.dtype == torch.float64 and np.isfinite(kl)
    assert [it for it, _ in timings.kl_history] == [100, 200, 300]
    e32, _, kl32 = bh.run(x.astype(np.float32),
                          bh.TsneConfig(n_iter=300, exaggeration_iters=100))
    # different precisions take different (chaotic) paths to similar optima
    assert abs(kl - kl32) / kl32 < 0.03


def test_sharded_engine_f64_single_rank_matches_unsharded(bh):
    import os
    import socket

    import torch.distributed as dist

    from paper_2212_11506_b200.dist import Shard
    g = golden("affinity450f64")
    p = bh.from_csr(g["row_offsets"], g["col_indices"], g["values"])
    y0 = np.column_stack([g["y0_init"], g["y1_init"]])
    cfg = bh.TsneConfig(n_iter=60, exaggeration_iters=20, graph_chunk=10,
                        precision="f64")
    e1 = bh.embedding_from(y0)
    bh.Engine(p, e1, cfg).run(60)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        e2 = bh.embedding_from(y0)
        bh.Engine(p, e2, cfg, shard=Shard(0, 1)).run(60)
    finally:
        dist.destroy_process_group()
    np.testing.assert_array_equal(e2.y.cpu().numpy(), e1.y.cpu().numpy())
