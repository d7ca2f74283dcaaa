"""GPU parity: every stage of the CUDA path against the CPU oracle and the
reference's golden vectors, through the C ABI.

Tolerances (north star): Morton codes, permutation, tree topology, masses
and centres of mass bit-exact; per-iteration gradients <= 1e-4 relative L2;
BSP betas <= 1e-5 relative; final KL within 1%.
"""

import zlib

import numpy as np
import pytest

from conftest import TREE_CASES, golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

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
    t = bh.summarize(bh.build_tree(mc, y))
    return (c, r), mc, t


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


# --- Morton / sort / tree: bit-exact against the reference goldens -------

@pytest.mark.parametrize("mode", [32, 64])
@pytest.mark.parametrize("case", TREE_CASES)
def test_tree_bit_exact_vs_reference_golden(bh, mode, case):
    g = golden(f"tree{mode}_{case}")
    y = g["y"]
    (c, r), mc, t = gpu_tree(bh, y, mode)
    assert c == tuple(g["center"]) and r == float(g["r_span"])
    ref_codes = g["codes"] if mode == 64 else g["codes"] >> np.uint64(32)
    np.testing.assert_array_equal(mc.codes_u64(), ref_codes)
    np.testing.assert_array_equal(mc.order.cpu().numpy(), g["order"])
    out = t.to_reference()
    for f in TOPO:
        np.testing.assert_array_equal(out[f], g[f], err_msg=f)


def test_golden_dump(bh):
    g = golden("tree64_dump4")
    _, _, t = gpu_tree(bh, g["y"], 64)
    assert t.dump() == str(g["dump"])


@pytest.mark.parametrize("mode", [32, 64])
@pytest.mark.parametrize("kind", ["gauss", "heavy", "dups", "tiny_spread"])
def test_tree_bit_exact_vs_oracle_large(bh, oracle, mode, kind):
    rng = np.random.default_rng(zlib.crc32(f"{mode}-{kind}".encode()))
    n = 120_000
    if kind == "gauss":
        y = rng.standard_normal((n, 2))
    elif kind == "heavy":
        c = rng.uniform(-50, 50, (100, 2))
        y = c[rng.integers(0, 100, n)] + rng.standard_t(2.0, (n, 2))
    elif kind == "dups":
        base = rng.standard_normal((n // 50, 2))
        y = base[rng.integers(0, n // 50, n)]
    else:
        y = 1e3 + rng.standard_normal((n, 2)) * 1e-5
    y = y.astype(np.float32)
    (c, r), mc, t = gpu_tree(bh, y, mode)
    assert (c, r) == oracle.compute_bounds(y)
    codes, order, sc = oracle.morton_codes(y, c, r, mode)
    np.testing.assert_array_equal(mc.codes_u64(), codes)
    np.testing.assert_array_equal(mc.order.cpu().numpy(), order)
    ot = oracle.tree_from_sorted(sc, order, y, c, r, mode)
    out = t.to_reference()
    for f in TOPO:
        np.testing.assert_array_equal(out[f], getattr(ot, f), err_msg=f)


@pytest.mark.parametrize("mode", [32, 64])
@pytest.mark.parametrize("kind", ["gauss", "heavy", "dups", "tiny_spread"])
@pytest.mark.parametrize("n", [120_000, 4096, 2049])
def test_prefix_summarize_matches_exact(bh, mode, kind, n):
    """The engine's f32 summarize from f64 prefix sums against the bit-exact
    level-by-level one: counts, child words and leaf centres bitwise;
    internal centres within 2 f32 spacings (f64 rounding only)."""
    rng = np.random.default_rng(zlib.crc32(f"{mode}-{kind}-{n}".encode()))
    if kind == "gauss":
        y = rng.standard_normal((n, 2))
    elif kind == "heavy":
        c = rng.uniform(-50, 50, (100, 2))
        y = c[rng.integers(0, 100, n)] + rng.standard_t(2.0, (n, 2))
    elif kind == "dups":
        base = rng.standard_normal((max(1, n // 50), 2))
        y = base[rng.integers(0, len(base), n)]
    else:
        y = 1e3 + rng.standard_normal((n, 2)) * 1e-5
    y = y.astype(np.float32)
    _, _, t = gpu_tree(bh, y, mode)
    a = t.arrays
    m = int(a.level_off[a.max_depth + 1].item())
    exact = a.node[:m].cpu().numpy().copy()
    a.summarize_prefix()
    torch.cuda.synchronize()
    pref = a.node[:m].cpu().numpy()
    np.testing.assert_array_equal(pref[:, 2:].view(np.uint32),
                                  exact[:, 2:].view(np.uint32))
    leaf = (exact[:, 3].view(np.uint32) & np.uint32(0x80000000)) != 0
    np.testing.assert_array_equal(pref[leaf, :2].view(np.uint32),
                                  exact[leaf, :2].view(np.uint32))
    # internal centres: within one f32 spacing of the true f64 mean of the
    # node's points (the reference's child-order sums of f32-rounded child
    # centres drift by up to ~one spacing per level, hence no bitwise check)
    ys = a.ys.cpu().numpy().astype(np.float64)
    S = np.concatenate([np.zeros((1, 2)), np.cumsum(ys, axis=0)])
    start = a.node_start[:m].cpu().numpy().astype(np.int64)[~leaf]
    end = a.leaf_end[:m].cpu().numpy().astype(np.int64)[~leaf]
    true = (S[end] - S[start]) / (end - start)[:, None]
    np.testing.assert_array_equal(end - start, pref[~leaf, 2].astype(np.int64))
    got = pref[~leaf, :2].astype(np.float64)
    d = np.abs(got - true)
    # one spacing of the f32 grid at the larger magnitude (a truth just
    # below a power of two may round up into the next binade)
    ulp = np.spacing(np.maximum(np.abs(true), np.abs(got)).astype(np.float32))
    assert (d <= ulp).all(), d.max()


@pytest.mark.parametrize("bits", [8, 17, 32, 42, 64])
def test_radix_sort_is_stable_argsort(bh, bits):
    from paper_2212_11506_b200 import _lib
    rng = np.random.default_rng(bits)
    n = 300_001
    hi = (1 << bits) - 1
    keys = rng.integers(0, min(hi, 2**63 - 1), n, dtype=np.int64).astype(np.uint64)
    keys[::7] = keys[0]  # heavy duplicates
    dt = np.uint32 if bits <= 32 else np.uint64
    keys = keys.astype(dt)
    kd = torch.from_numpy(keys.view(np.int32 if bits <= 32 else np.int64)).cuda()
    sk = torch.empty_like(kd)
    order = torch.empty(n, dtype=torch.int32, device="cuda")
    lib = _lib.load()
    ws = _lib.workspace(lib.bh_sort_workspace_bytes(n, bits))
    for _ in range(2):  # workspace reuse must leave counters at zero
        _lib.call("bh_sort", _lib.ptr(kd), n, bits, _lib.ptr(sk),
                  _lib.ptr(order), _lib.ptr(ws), ws.numel(), _lib.stream())
        ref = np.argsort(keys, kind="stable")
        np.testing.assert_array_equal(order.cpu().numpy(), ref)
        np.testing.assert_array_equal(sk.cpu().numpy().view(dt), keys[ref])


# --- forces ---------------------------------------------------------------

@pytest.mark.parametrize("mode", [32, 64])
@pytest.mark.parametrize("case", ["gauss2000", "heavy3200", "coinc7", "two",
                                  "quad4"])
@pytest.mark.parametrize("theta", [0.0, 0.5, 0.8])
def test_repulsive_vs_reference_golden(bh, mode, case, theta):
    g = golden(f"tree{mode}_{case}")
    y = g["y"]
    _, _, t = gpu_tree(bh, y, mode)
    buf = bh.GradientBuffers.allocate(y.shape[0])
    bh.repulsive_bh(t, y, theta, buf)
    tag = f"bh{int(theta * 10)}"
    ref = np.column_stack([g[tag + "_rep0"], g[tag + "_rep1"]])
    got = buf.rep.cpu().numpy()
    # f32 pair math vs the reference's f64: per-point relative error
    norm = np.linalg.norm(ref, axis=1)
    err = np.linalg.norm(got - ref, axis=1)
    assert (err <= 2e-5 * np.maximum(norm, 1e-3 * norm.max()) + 1e-30).all()
    np.testing.assert_allclose(buf.z_partial.cpu().numpy(), g[tag + "_zpart"],
                               rtol=2e-6)
    assert buf.z == pytest.approx(float(g[tag + "_z"]), rel=1e-6)


@pytest.mark.parametrize("mode", [32, 64])
def test_repulsive_large_vs_oracle(bh, oracle, mode):
    rng = np.random.default_rng(3)
    c = rng.uniform(-50, 50, (100, 2))
    y = (c[rng.integers(0, 100, 200_000)]
         + rng.standard_t(2.0, (200_000, 2))).astype(np.float32)
    _, _, t = gpu_tree(bh, y, mode)
    buf = bh.GradientBuffers.allocate(y.shape[0])
    bh.repulsive_bh(t, y, 0.5, buf)
    ot = oracle.build_tree(y, code_bits=mode)
    r0, r1, zp, z = oracle.repulsive_bh(ot, y, 0.5)
    ref = np.column_stack([r0, r1])
    assert rel_l2(buf.rep.cpu().numpy(), ref) < 1e-5
    assert buf.z == pytest.approx(z, rel=1e-7)
    cnt = bh.repulsive_counts(t, 0.5)
    _, _, _, _, oc = oracle.repulsive_bh(ot, y, 0.5, counts=True)
    # per-point visit counts equal the reference traversal's (exact BH
    # semantics of the warp-synchronous walk); f32 vs f64 accept decisions
    # may flip on a handful of boundary cases
    mism = (cnt[:, 0] != oc[:, 0]).mean()
    assert mism < 1e-3
    assert abs(cnt[:, 0].sum() - oc[:, 0].sum()) / oc[:, 0].sum() < 1e-4


def test_repulsive_theta0_equals_exact(bh):
    rng = np.random.default_rng(11)
    y = rng.standard_normal((500, 2)).astype(np.float32)
    _, _, t = gpu_tree(bh, y, 32)
    bhb = bh.GradientBuffers.allocate(500)
    bh.repulsive_bh(t, y, 0.0, bhb)
    ex = bh.GradientBuffers.allocate(500)
    bh.repulsive_exact(y, ex)
    assert rel_l2(bhb.rep.cpu().numpy(), ex.rep.cpu().numpy()) < 1e-6
    assert bhb.z == pytest.approx(ex.z, rel=1e-7)


def test_attractive_vs_reference_golden(bh):
    g = golden("affinity450")
    p = bh.from_csr(g["row_offsets"], g["col_indices"], g["values"])
    for fac, a0, a1 in ((1.0, "attr0", "attr1"), (12.0, "attr12_0", "attr12_1")):
        buf = bh.GradientBuffers.allocate(450)
        bh.attractive(bh.set_exaggeration(p, fac), g["y"], buf)
        ref = np.column_stack([g[a0], g[a1]])
        assert rel_l2(buf.attr.cpu().numpy(), ref) < 1e-6


def test_attractive_two_point_and_empty_row(bh):
    p = bh.from_csr([0, 1, 2, 2], [1, 0], np.array([0.5, 0.5], np.float32))
    y = np.array([[0.0, 0.0], [1.0, 0.0], [5.0, 5.0]], np.float32)
    buf = bh.GradientBuffers.allocate(3)
    bh.attractive(p, y, buf)
    np.testing.assert_allclose(buf.attr.cpu().numpy(),
                               [[-0.25, 0.0], [0.25, 0.0], [0.0, 0.0]],
                               atol=1e-7)
    with pytest.raises(ValueError, match="matrix is over 3 points"):
        bh.attractive(p, y[:2], buf)


# --- affinities -----------------------------------------------------------

def test_bsp_and_symmetrize_vs_reference_golden(bh):
    g = golden("affinity450")
    graph = bh.NeighborGraph(g["indices"], g["sq_distances"])
    pr = bh.calibrate_perplexity(graph, 10.0)
    betas = pr.betas.cpu().numpy()
    assert np.max(np.abs(betas - g["betas"]) / g["betas"]) <= 1e-5
    np.testing.assert_allclose(pr.conditional.cpu().numpy(), g["cond"],
                               rtol=1e-9, atol=1e-300)
    p = bh.symmetrize(pr, graph)
    ro, co, va = p.to_reference()
    np.testing.assert_array_equal(ro, g["row_offsets"])
    np.testing.assert_array_equal(co, g["col_indices"])
    # values: same f64 sums, cast to f32 -> equal up to one f32 ulp
    np.testing.assert_allclose(va, g["values"], rtol=1.2e-7, atol=0)
    # symmetric with bitwise-equal values (test_affinity.py:148-164)
    rows = np.repeat(np.arange(450), np.diff(ro))
    d = {(r, c): v for r, c, v in zip(rows, co, va)}
    assert all(d[(c, r)] == v for (r, c), v in d.items())


def test_symmetrize_exact_from_reference_conditionals(bh):
    """Fed the reference's own conditionals, the CSR is bit-identical."""
    g = golden("affinity450")
    graph = bh.NeighborGraph(g["indices"], g["sq_distances"])
    from paper_2212_11506_b200.affinity import PerplexityResult
    pr = PerplexityResult(betas=torch.from_numpy(g["betas"]).cuda(),
                          conditional=torch.from_numpy(g["cond"]).cuda())
    ro, co, va = bh.symmetrize(pr, graph).to_reference()
    np.testing.assert_array_equal(va, g["values"])


def test_bsp_edge_cases(bh):
    g = bh.NeighborGraph(np.array([[1, 2]]), np.array([[4.0, 4.0]]))
    pr = bh.calibrate_perplexity(g, 2.0)
    np.testing.assert_array_equal(pr.conditional.cpu().numpy()[0], [0.5, 0.5])
    g = bh.NeighborGraph(np.array([[1, 2, 3]]), np.zeros((1, 3)))
    pr = bh.calibrate_perplexity(g, 2.0)
    np.testing.assert_allclose(pr.conditional.cpu().numpy()[0], 1 / 3)
    with pytest.raises(ValueError, match="perplexity exceeds neighborhood"):
        bh.calibrate_perplexity(bh.NeighborGraph(np.array([[1, 2]]),
                                                 np.array([[1.0, 2.0]])), 3.0)


def test_knn_exact_vs_reference(bh):
    from paper_2212_11506_b200.knn import knn_exact
    g = golden("affinity450")
    kg = knn_exact(g["x"], 30)
    np.testing.assert_array_equal(kg.indices.cpu().numpy(), g["indices"])
    np.testing.assert_array_equal(kg.sq_distances.cpu().numpy(),
                                  g["sq_distances"])
    from paper_2212_11506_b200.workloads import c0
    kg = knn_exact(c0(), 90)
    np.testing.assert_array_equal(kg.indices.cpu().numpy(),
                                  golden("c0_run")["indices"].astype(np.int64))


@pytest.mark.parametrize("n,d,k", [(600, 100, 40), (700, 12, 200),
                                   (300, 784, 299), (1500, 50, 150),
                                   (333, 64, 332), (900, 7, 600)])
def test_knn_general_any_d_and_k(bh, oracle, n, d, k):
    """Beyond bh_knn's D <= 64 / k <= 128 (e.g. perplexity 50+, raw
    784-pixel images): bh_knn_general, the same semantics (f64 column-order
    sums, ties -> lower id) against the oracle's knn.py restatement.
    float32 rows of D <= 64 take the tile filter with its lists in the
    scratch (any k); wider rows and float64 the streaming kernel."""
    from paper_2212_11506_b200.knn import knn_exact
    rng = np.random.default_rng(d)
    x = rng.integers(0, 4, (n, d)).astype(np.float32)  # many exact ties
    for dt in (np.float32, np.float64):
        g = knn_exact(x.astype(dt), k)
        idx, sqd = oracle.knn_exact(x.astype(dt), k)
        np.testing.assert_array_equal(g.indices.cpu().numpy(), idx)
        np.testing.assert_array_equal(g.sq_distances.cpu().numpy(), sqd)


# --- optimiser ------------------------------------------------------------

def test_gradient_step_trajectory_vs_reference(bh):
    """Eight reference gradient_step calls (exaggerated, then across the
    momentum switch) on the same P: gradients match to <= 1e-4 rel-L2 at
    every step, so the trajectories stay together."""
    a = golden("affinity450")
    g = golden("trajectory450")
    p = bh.from_csr(a["row_offsets"], a["col_indices"], a["values"])
    pe = bh.set_exaggeration(p, 12.0)
    e = bh.embedding_from(np.column_stack([g["y0_init"], g["y1_init"]]))
    cfg = bh.TsneConfig(perplexity=10.0, code_bits=64)
    for it in range(8):
        if it == 4:
            e.iteration = 250
        bh.gradient_step(e, pe if it < 4 else p, cfg)
        ref = np.column_stack([g[f"y0_{it}"], g[f"y1_{it}"]])
        assert rel_l2(e.y.cpu().numpy(), ref) < 1e-5, it


@pytest.mark.parametrize("code_bits", [32, 64])
def test_gradient_parity_late_iterations(bh, oracle, code_bits):
    """Run the oracle to iterations {0, 250, 500, 999} of the C0 schedule and
    compare the GPU gradient on the same Y snapshot (rel-L2 <= 1e-4)."""
    from paper_2212_11506_b200.workloads import c0
    x = c0()
    idx, sqd = oracle.knn_exact(x, 90)
    betas, cond = oracle.calibrate_perplexity(sqd, 30.0)
    ro, co, va = oracle.symmetrize(idx, cond)
    p = bh.from_csr(ro, co, va)
    s = oracle.State.init(2048, 0)
    checkpoints = {0, 250, 500, 999}
    for it in range(1000):
        vals = oracle.exaggerate(va, 12.0) if it < 250 else va
        if it in checkpoints:
            y = np.column_stack([s.y0, s.y1])
            g0, g1, _, _, _ = oracle.gradient(y, ro, co, vals, 0.5, code_bits)
            ref = np.column_stack([g0, g1])
            pp = bh.set_exaggeration(p, 12.0 if it < 250 else 1.0)
            (c, r), mc, t = gpu_tree(bh, y, code_bits)
            buf = bh.GradientBuffers.allocate(2048)
            bh.attractive(pp, y, buf)
            bh.repulsive_bh(t, y, 0.5, buf)
            zf = np.float32(buf.z)
            got = np.float32(4.0) * (buf.attr.cpu().numpy()
                                     - buf.rep.cpu().numpy() / zf)
            assert rel_l2(got, ref) <= 1e-4, (it, rel_l2(got, ref))
        oracle.gradient_step(s, ro, co, vals, code_bits=code_bits)


def test_engine_graph_equals_eager_and_is_deterministic(bh):
    a = golden("affinity450")
    p = bh.from_csr(a["row_offsets"], a["col_indices"], a["values"])
    outs = []
    for use_graph in (True, True, False):
        e = bh.init_embedding(450, seed=3)
        cfg = bh.TsneConfig(n_iter=60, exaggeration_iters=20, graph_chunk=7)
        eng = bh.Engine(p, e, cfg)
        eng.run(60, use_graph=use_graph)
        outs.append(e.y.cpu().numpy().copy())
    np.testing.assert_array_equal(outs[0], outs[1])
    np.testing.assert_array_equal(outs[0], outs[2])


@pytest.mark.parametrize("code_bits,theta", [(32, 0.5), (64, 0.5), (32, 0.8)])
def test_fused_forces_bitwise_equal_separate(bh, code_bits, theta):
    """bh_forces (one launch, interleaved traversal and CSR-sweep CTAs) gives
    the bitwise trajectory of the separate attractive + repulsive kernels,
    in the fast path and in the evented path."""
    rng = np.random.default_rng(5)
    n, k = 30_000, 24
    col = rng.integers(0, n - 1, (n, k))
    col += col >= np.arange(n)[:, None]  # no self edges
    val = rng.uniform(0.1, 1.0, (n, k)).astype(np.float32)
    val /= val.sum()
    p = bh.from_csr(np.arange(0, n * k + 1, k), col.ravel().astype(np.int32),
                    val.ravel())
    y0 = rng.standard_normal((n, 2)).astype(np.float32)
    outs = []
    for fuse, timed in ((True, False), (False, False), (True, True)):
        e = bh.embedding_from(y0)
        cfg = bh.TsneConfig(n_iter=60, exaggeration_iters=20, graph_chunk=10,
                            code_bits=code_bits, relabel_every=20,
                            theta=theta)
        eng = bh.Engine(p, e, cfg)
        eng.fuse = fuse
        eng.fuse_timed = timed
        tm = bh.StepTimings() if timed else None
        eng.run(60, tm)
        if timed:
            assert tm.calls("forces") == 60 and tm.calls("repulsive") == 0
        outs.append(e.y.cpu().numpy().copy())
    np.testing.assert_array_equal(outs[0], outs[1])
    np.testing.assert_array_equal(outs[0], outs[2])


def test_non_finite_gradient_reports_point(bh):
    p = bh.from_csr([0, 1, 2], [1, 0], np.array([0.5, 0.5], np.float32))
    e = bh.embedding_from(np.array([[-1e30, 0.0], [1e30, 0.0]], np.float32))
    with pytest.raises(ValueError, match="non-finite gradient at point 0"):
        bh.gradient_step(e, p, bh.TsneConfig(n_iter=10, exaggeration_iters=0))


def test_recentred_and_momentum_switch(bh):
    p = bh.from_csr([0, 1, 2], [1, 0], np.array([0.5, 0.5], np.float32))
    for it, mom in ((249, 0.5), (250, 0.8)):
        e = bh.embedding_from(np.array([[-0.5, 0.0], [0.5, 0.0]], np.float32),
                              v=np.array([[0.02, 0.0], [-0.01, 0.0]], np.float32))
        e.iteration = it
        v_before = e.v.cpu().numpy().copy()
        bh.gradient_step(e, p, bh.TsneConfig(n_iter=300, theta=0.0))
        np.testing.assert_allclose(e.v.cpu().numpy()[:, 0],
                                   mom * v_before[:, 0], atol=1e-7)
        assert abs(float(e.y[:, 0].double().mean())) < 1e-7


@pytest.mark.slow
def test_c0_full_run_kl_within_1pct(bh):
    from paper_2212_11506_b200.workloads import c0
    g = golden("c0_run")
    knn = (g["indices"].astype(np.int64), None)
    from oracle import oracle as o
    idx, sqd = o.knn_exact(c0(), 90)
    e, timings, kl = bh.run(c0(), bh.TsneConfig(kl_every=250),
                            knn=(idx, sqd))
    # one chaotic trajectory: its final KL must fall inside the spread of the
    # reference's own runs over Y0 seeds 0..7 (widened by 1%); the 1%
    # criterion itself is checked on the 8-seed median below
    ref = golden("c0_seeds")["kl"].astype(np.float64)
    assert float(g["kl"]) == ref[0]
    assert 0.99 * ref.min() < kl < 1.01 * ref.max(), kl
    assert timings.calls("tree") == 1000
    assert [it for it, _ in timings.kl_history] == [250, 500, 750, 1000]
    # and through the GPU kNN (run without a graph)
    e2, _, kl2 = bh.run(c0(), bh.TsneConfig())
    np.testing.assert_array_equal(e2.y.cpu().numpy(), e.y.cpu().numpy())


@pytest.mark.slow
def test_c0_seed_median_kl_within_1pct(bh):
    """The trajectory is chaotic: any change of f32 summation order gives
    another, equally valid one (the reference's own final KL over Y0 seeds
    0..7 spans 1.6565..1.6815).  The 1% criterion on a statistic that does
    not hinge on one trajectory: the median final KL over the same 8 seeds,
    ours against the unmodified reference's (tests/golden c0_seeds)."""
    from paper_2212_11506_b200.workloads import c0
    from oracle import oracle as o
    ref = golden("c0_seeds")["kl"].astype(np.float64)
    x = c0()
    idx, sqd = o.knn_exact(x, 90)
    ours = [bh.run(x, bh.TsneConfig(seed=s), knn=(idx, sqd))[2]
            for s in range(len(ref))]
    med_o, med_r = float(np.median(ours)), float(np.median(ref))
    assert abs(med_o - med_r) / med_r < 0.01, (ours, ref.tolist())
    # every one of our runs inside the reference's seed range, widened by 1%
    assert min(ours) > 0.99 * ref.min() and max(ours) < 1.01 * ref.max(), ours


@pytest.mark.slow
def test_c1_full_run_kl_within_1pct(bh):
    """C1 (N=70k, D=50): the whole pipeline from raw data on the GPU (exact
    kNN, BSP, P, Y0, 1000 iterations, exact KL) against the unmodified
    reference's run() on the same data (tests/golden c1_run)."""
    from paper_2212_11506_b200.workloads import c1
    g = golden("c1_run")
    e, timings, kl = bh.run(c1(), bh.TsneConfig(kl_every=250))
    ref = float(g["kl"])
    assert abs(kl - ref) / ref < 0.01, (kl, ref)
    ours = [k for _, k in timings.kl_history]
    theirs = [float(k) for _, k in g["kl_history"]]
    assert len(ours) == len(theirs) == 4
    # the periodic BH-KL follows the same descent
    assert all(abs(a - b) / b < 0.05 for a, b in zip(ours, theirs)), (ours, theirs)


@pytest.mark.slow
def test_c2_full_run_kl_within_1pct(bh):
    """C2 (N=250k, D=50, 20 rotated anisotropic clusters): the whole GPU
    pipeline from raw data against the unmodified reference's run()."""
    from paper_2212_11506_b200.workloads import c2
    g = golden("c2_run")
    e, timings, kl = bh.run(c2(), bh.TsneConfig(kl_every=250))
    ref = float(g["kl"])
    assert abs(kl - ref) / ref < 0.01, (kl, ref)
    ours = [k for _, k in timings.kl_history]
    theirs = [float(k) for _, k in g["kl_history"]]
    assert all(abs(a - b) / b < 0.05 for a, b in zip(ours, theirs)), (ours, theirs)


@pytest.mark.parametrize("n", [3, 5, 17, 33, 129, 300])
def test_small_sizes_through_run(bh, n):
    """Ragged sizes (partial warps / CTAs, fewer rows than one sweep batch,
    side-sweep split of 0 or 1 rows) through the whole public pipeline,
    against the same run with separate force kernels."""
    rng = np.random.default_rng(n)
    x = rng.standard_normal((n, 4)).astype(np.float32)
    cfg = bh.TsneConfig(perplexity=min(30.0, (n - 1) / 3.0 + 0.5), n_iter=60,
                        exaggeration_iters=20, relabel_every=7, graph_chunk=5)
    e, timings, kl = bh.run(x, cfg)
    y = e.y.cpu().numpy()
    assert y.shape == (n, 2) and np.isfinite(y).all() and np.isfinite(kl)
    assert timings.calls("tree") == 60
    # the engine's separate-kernel path gives the bitwise same trajectory
    from paper_2212_11506_b200.optimizer import affinities
    p, _ = affinities(x, cfg)
    e2 = bh.init_embedding(n, cfg.seed)
    eng = bh.Engine(p, e2, cfg)
    eng.fuse = False
    eng.run(60)
    np.testing.assert_array_equal(e2.y.cpu().numpy(), y)


def test_estimator_fit_transform(bh):
    from paper_2212_11506_b200.workloads import c0
    est = bh.BarnesHutTSNE(n_iter=300, exaggeration_iters=100)
    y = est.fit_transform(c0()[:1024])
    assert y.shape == (1024, 2) and np.isfinite(y).all()
    assert est.kl_divergence_ > 0 and est.manifest_["kl"] == est.kl_divergence_
    assert est.timings_["tree"]["calls"] == 300


def test_sharded_engine_single_rank_matches_unsharded(bh):
    """The multi-GPU code path (Shard: row/position ranges, sorted-order
    forces, NCCL all-gathers, Z partials) on a 1-rank NCCL group must give
    the bitwise-identical trajectory of the unsharded engine."""
    import os
    import socket

    import torch.distributed as dist

    from paper_2212_11506_b200.dist import Shard
    a = golden("affinity450")
    p = bh.from_csr(a["row_offsets"], a["col_indices"], a["values"])
    cfg = bh.TsneConfig(n_iter=80, exaggeration_iters=30, graph_chunk=10)
    e1 = bh.init_embedding(450, seed=3)
    bh.Engine(p, e1, cfg).run(80)
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        e2 = bh.init_embedding(450, seed=3)
        bh.Engine(p, e2, cfg, shard=Shard(0, 1)).run(80)
    finally:
        dist.destroy_process_group()
    np.testing.assert_array_equal(e2.y.cpu().numpy(), e1.y.cpu().numpy())


def test_checkpoint_resume_continues_the_schedule(bh, tmp_path):
    """Embedding.save / load: 40 iterations, a checkpoint, 40 more from the
    restored state (across the exaggeration switch at 50) equal 80 straight
    iterations bit for bit (relabel off: both runs keep the id order)."""
    a = golden("affinity450")
    p = bh.from_csr(a["row_offsets"], a["col_indices"], a["values"])
    cfg = bh.TsneConfig(n_iter=80, exaggeration_iters=50, graph_chunk=10,
                        relabel_every=0)
    e1 = bh.init_embedding(450, seed=5)
    bh.Engine(p, e1, cfg).run(80)
    e2 = bh.init_embedding(450, seed=5)
    bh.Engine(p, e2, cfg).run(40)
    e2.save(tmp_path / "ck.npz")
    e3 = bh.Embedding.load(tmp_path / "ck.npz")
    assert e3.iteration == 40
    bh.Engine(p, e3, cfg).run(40)
    np.testing.assert_array_equal(e3.y.cpu().numpy(), e1.y.cpu().numpy())
    assert e3.iteration == 80
