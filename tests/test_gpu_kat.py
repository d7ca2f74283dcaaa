"""Known-answer and invariant tests of the reference's own test suite
(pkg/tests: test_quadtree.py, test_forces.py, test_affinity.py,
test_optimizer.py, test_acceptance.py -- SURVEY.md 8(c)), restated against
the CUDA path through the public API.  The reference runs these in its
default float64 precision; so do they here (the `_f64` kernels), with the
reference's tolerances.
"""

import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bh():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2212_11506_b200 as m
    return m


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


def make_tree(bh, y, code_bits=64):
    c, r = bh.compute_bounds(y, code_bits)
    mc = bh.morton_codes(y, c, r, code_bits)
    t = bh.summarize(bh.build_tree(mc, y))
    return mc, t, t.to_reference()


# --- quadtree (test_quadtree.py:164-288) ----------------------------------

@pytest.mark.parametrize("code_bits", [32, 64])
def test_tree_structure_invariants(bh, rng, code_bits):
    n = 1500
    y = rng.standard_normal((n, 2))
    mc, t, r = make_tree(bh, y, code_bits)
    lo, start, end, ch = r["level_offsets"], r["start"], r["end"], r["children"]
    leaf, depth = r["is_leaf"].astype(bool), r["depth"]
    D = code_bits // 2
    assert lo[0] == 0 and lo[-1] == t.n_nodes and (np.diff(lo) > 0).all()
    assert (start[0], end[0]) == (0, n)
    for nd in range(t.n_nodes):
        cnt = end[nd] - start[nd]
        if leaf[nd]:
            assert (ch[nd] == -1).all()
            assert cnt == 1 or depth[nd] == D      # leaf rule
            continue
        assert cnt > 1
        kids = ch[nd][ch[nd] >= 0]
        assert len(kids) >= 1 and (depth[kids] == depth[nd] + 1).all()
        assert (np.sort(kids) == kids).all()
        # children partition the parent's point range
        assert start[kids[0]] == start[nd] and end[kids[-1]] == end[nd]
        assert (end[kids[:-1]] == start[kids[1:]]).all()
    # leaves partition the points
    cover = np.zeros(n, int)
    for nd in np.flatnonzero(leaf):
        cover[start[nd]:end[nd]] += 1
    assert (cover == 1).all()
    # a node's points are exactly the codes sharing its prefix
    sc = r["sorted_codes"]
    width = 2 * D
    for nd in range(1, t.n_nodes, 7):
        shift = np.uint64(width - 2 * depth[nd])
        pre = sc[start[nd]] >> shift
        match = (sc >> shift) == pre
        assert match.sum() == end[nd] - start[nd]
        assert match[start[nd]:end[nd]].all()
    # the cell radius halves per level
    np.testing.assert_array_equal(r["cell_radius"], t.r_span / 2.0 ** depth)


@pytest.mark.parametrize("code_bits", [32, 64])
def test_coincident_points_aggregate_at_max_depth(bh, code_bits):
    y = np.array([[1.0, 1.0]] * 5 + [[-1.0, -1.0]] * 2)
    _, t, r = make_tree(bh, y, code_bits)
    assert t.n_levels == code_bits // 2 + 1
    leaves = np.flatnonzero(r["is_leaf"])
    assert sorted(r["mass"][leaves].tolist()) == [2, 5]
    assert r["mass"][0] == 7


def test_summary_leaf_root_slices_and_telescoping(bh, rng):
    # leaf mass 1 with com = the point itself
    y = rng.standard_normal((100, 2))
    mc, t, r = make_tree(bh, y)
    order = mc.order.cpu().numpy()
    for nd in np.flatnonzero(r["is_leaf"]):
        if r["end"][nd] - r["start"][nd] == 1:
            assert r["mass"][nd] == 1
            np.testing.assert_array_equal(r["com"][nd], y[order[r["start"][nd]]])
    # root = mean
    y = rng.standard_normal((2048, 2))
    _, _, r = make_tree(bh, y)
    assert r["mass"][0] == 2048
    np.testing.assert_allclose(r["com"][0], y.mean(axis=0), atol=1e-12)
    # every node's com is the mean of its slice, mass its size
    y = rng.random((1000, 2))
    mc, t, r = make_tree(bh, y)
    ys = y[mc.order.cpu().numpy()]
    for nd in range(t.n_nodes):
        s, e = r["start"][nd], r["end"][nd]
        np.testing.assert_allclose(r["com"][nd], ys[s:e].mean(axis=0),
                                   rtol=1e-12, atol=1e-14)
        assert r["mass"][nd] == e - s
    # mass telescopes: leaves above a level plus the level's nodes hold all
    y = rng.standard_normal((512, 2))
    _, t, r = make_tree(bh, y)
    leaf, depth = r["is_leaf"].astype(bool), r["depth"]
    for lvl in range(t.n_levels):
        front = (depth == lvl) | (leaf & (depth < lvl))
        assert r["mass"][front].sum() == 512


# --- repulsion (test_forces.py:150-235) -------------------------------------

def _forces(bh, y, theta):
    _, t, _ = make_tree(bh, y)
    b = bh.GradientBuffers.allocate(y.shape[0], np.float64)
    bh.repulsive_bh(t, y, theta, b)
    return b


def _exact(bh, y):
    b = bh.GradientBuffers.allocate(y.shape[0], np.float64)
    bh.repulsive_exact(y, b)
    return b


def test_bh_two_points_closed_form(bh):
    y = np.array([[0.0, 0.0], [0.0, 3.0]])
    b = _forces(bh, y, 0.5)
    assert b.z == pytest.approx(2.0 / 10.0, rel=1e-15)
    np.testing.assert_allclose(b.rep.cpu().numpy()[0], [0.0, -3.0 / 100.0],
                               rtol=1e-15)


def test_bh_theta0_equals_exact(bh, rng):
    y = rng.standard_normal((500, 2))
    b, ex = _forces(bh, y, 0.0), _exact(bh, y)
    np.testing.assert_allclose(b.z_partial.cpu().numpy(),
                               ex.z_partial.cpu().numpy(), rtol=1e-10)
    assert abs(b.z - ex.z) / ex.z < 1e-10
    er, gr = ex.rep.cpu().numpy(), b.rep.cpu().numpy()
    norm = np.linalg.norm(er, axis=1)
    err = np.linalg.norm(gr - er, axis=1)
    assert (err <= 1e-10 * np.maximum(norm, 1e-3 * norm.max())).all()


def test_bh_accuracy_theta_half(bh, rng):
    y = rng.standard_normal((2000, 2))
    b, ex = _forces(bh, y, 0.5), _exact(bh, y)
    er = ex.rep.cpu().numpy()
    rel = np.linalg.norm(b.rep.cpu().numpy() - er, axis=1) / np.linalg.norm(er, axis=1)
    assert np.percentile(rel, 95) <= 0.02
    assert abs(b.z - ex.z) / ex.z <= 0.005


def test_bh_error_monotone_in_theta(bh, rng):
    y = rng.standard_normal((1200, 2))
    _, t, _ = make_tree(bh, y)
    er = _exact(bh, y).rep.cpu().numpy()
    norm = np.linalg.norm(er, axis=1)
    means = []
    for theta in (0.8, 0.5, 0.2, 0.0):
        b = bh.GradientBuffers.allocate(1200, np.float64)
        bh.repulsive_bh(t, y, theta, b)
        means.append((np.linalg.norm(b.rep.cpu().numpy() - er, axis=1) / norm).mean())
    assert means[0] >= means[1] >= means[2] >= means[3]


def test_bh_requires_summarized_tree(bh, rng):
    y = rng.standard_normal((50, 2))
    mc = bh.morton_codes(y, *bh.compute_bounds(y))
    t = bh.build_tree(mc, y)
    with pytest.raises(ValueError, match="summarized"):
        bh.repulsive_bh(t, y, 0.5, bh.GradientBuffers.allocate(50, np.float64))


def test_coincident_points_z_contribution(bh):
    # coincident points exert no force on each other but count in z
    y = np.array([[1.0, 1.0], [1.0, 1.0], [-1.0, -1.0]])
    b, ex = _forces(bh, y, 0.5), _exact(bh, y)
    zp = b.z_partial.cpu().numpy()
    np.testing.assert_allclose(zp, ex.z_partial.cpu().numpy(), rtol=1e-12)
    assert zp[0] == pytest.approx(1.0 + 1.0 / 9.0, rel=1e-12)


# --- affinities (test_affinity.py:44-176) -----------------------------------

def _graph(bh, sqd):
    sqd = np.asarray(sqd, np.float64)
    n, k = sqd.shape
    idx = (np.arange(n)[:, None] + 1 + np.arange(k)[None, :]) % max(n, k + 1)
    return bh.NeighborGraph(idx, sqd)


def _entropy_bits(p):
    p = p[p > 0]
    return float(-(p * np.log2(p)).sum())


def _beta_oracle(row, u, iters=200):
    """Independent bisection on beta: the Gaussian kernel over the shifted
    distances whose perplexity 2^H equals u."""
    d = np.asarray(row, np.float64) - min(row)
    lo, hi = 0.0, 1e6
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        w = np.exp(-mid * d)
        p = w / w.sum()
        if 2.0 ** _entropy_bits(p) > u:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def test_bsp_known_answers(bh, rng):
    pr = bh.calibrate_perplexity(_graph(bh, [[4.0, 4.0]]), 2.0)
    cond = pr.conditional.cpu().numpy()[0]
    np.testing.assert_array_equal(cond, [0.5, 0.5])
    assert _entropy_bits(cond) == 1.0
    row = [1.0, 4.0, 9.0]
    pr = bh.calibrate_perplexity(_graph(bh, [row]), 2.0, tol=1e-10)
    expect = _beta_oracle(row, 2.0)
    assert abs(float(pr.betas[0]) - expect) / expect < 1e-6
    sqd = np.sort(rng.random((50, 8)) * 5, axis=1)
    pr = bh.calibrate_perplexity(_graph(bh, sqd), 4.0)
    np.testing.assert_allclose(pr.conditional.cpu().numpy().sum(axis=1), 1.0,
                               atol=1e-12)
    assert (pr.betas.cpu().numpy() > 0).all()
    pr = bh.calibrate_perplexity(_graph(bh, [[0.0, 0.0, 0.0]]), 2.0)
    np.testing.assert_allclose(pr.conditional.cpu().numpy()[0], 1.0 / 3.0)
    assert float(pr.betas[0]) > 0
    with pytest.raises(ValueError, match="perplexity exceeds neighborhood"):
        bh.calibrate_perplexity(_graph(bh, [[1.0, 2.0]]), 3.0)
    with pytest.raises(ValueError, match="> 1"):
        bh.calibrate_perplexity(_graph(bh, [[1.0, 2.0]]), 1.0)


def test_perplexity_hits_target(bh, rng):
    from paper_2212_11506_b200.knn import knn_exact
    data = rng.standard_normal((300, 8))
    g = knn_exact(data, 40)
    cond = bh.calibrate_perplexity(g, 12.0).conditional.cpu().numpy()
    for i in range(300):
        assert abs(2.0 ** _entropy_bits(cond[i]) - 12.0) / 12.0 <= 1e-4


def _dense(p):
    ro, co, va = p.to_reference()
    d = np.zeros((p.n, p.n))
    for i in range(p.n):
        d[i, co[ro[i]:ro[i + 1]]] = va[ro[i]:ro[i + 1]]
    return d


def test_symmetrize_closed_forms(bh):
    from paper_2212_11506_b200.affinity import PerplexityResult
    dev = torch.device("cuda")
    ones = lambda n: PerplexityResult(
        betas=torch.ones(n, dtype=torch.float64, device=dev),
        conditional=torch.ones((n, 1), dtype=torch.float64, device=dev))
    g = bh.NeighborGraph(np.array([[1], [0]]), np.ones((2, 1)))
    p = bh.symmetrize(ones(2), g, dtype=np.float64)
    np.testing.assert_array_equal(_dense(p), [[0.0, 0.5], [0.5, 0.0]])
    assert float(p.base_values.sum()) == pytest.approx(1.0, abs=1e-15)
    # one-sided contributions: 0 -> 1, 1 -> 2, 2 -> 1
    g = bh.NeighborGraph(np.array([[1], [2], [1]]), np.ones((3, 1)))
    d = _dense(bh.symmetrize(ones(3), g, dtype=np.float64))
    assert d[0, 1] == pytest.approx(1 / 6) and d[1, 0] == d[0, 1]
    assert d[1, 2] == pytest.approx(2 / 6)
    np.testing.assert_array_equal(d, d.T)


def test_symmetrize_dense_oracle_and_csr_invariants(bh, rng):
    from paper_2212_11506_b200.knn import knn_exact
    data = rng.standard_normal((50, 4))
    g = knn_exact(data, 10)
    pr = bh.calibrate_perplexity(g, 5.0)
    p = bh.symmetrize(pr, g, dtype=np.float64)
    n, k = 50, 10
    cond = np.zeros((n, n))
    idx = g.indices.cpu().numpy()
    cc = pr.conditional.cpu().numpy()
    for i in range(n):
        cond[i, idx[i]] = cc[i]
    np.testing.assert_allclose(_dense(p), (cond + cond.T) / (2.0 * n),
                               rtol=1e-13, atol=1e-18)
    data = rng.standard_normal((80, 5))
    g = knn_exact(data, 12)
    p = bh.symmetrize(bh.calibrate_perplexity(g, 6.0), g, dtype=np.float64)
    ro, co, va = p.to_reference()
    assert ro[0] == 0 and ro[-1] == p.nnz and (np.diff(ro) >= 0).all()
    assert (va > 0).all() and abs(va.sum() - 1.0) < 1e-10
    rows = np.repeat(np.arange(p.n), np.diff(ro))
    assert not (rows == co).any()
    ent = {(int(r), int(c)): v for r, c, v in zip(rows, co, va)}
    assert all((c, r) in ent and ent[(c, r)] == v for (r, c), v in ent.items())


def test_exaggeration_roundtrip_bitwise(bh, rng):
    from paper_2212_11506_b200.knn import knn_exact
    g = knn_exact(rng.standard_normal((40, 4)), 8)
    p = bh.symmetrize(bh.calibrate_perplexity(g, 4.0), g, dtype=np.float64)
    orig = p.values.cpu().numpy().copy()
    p12 = bh.set_exaggeration(p, 12.0)
    assert abs(float(p12.values.sum()) - 12.0) < 1e-12 and p12.exaggeration == 12.0
    np.testing.assert_array_equal(bh.set_exaggeration(p12, 1.0).values.cpu().numpy(),
                                  orig)


# --- attraction (test_forces.py:54-84) --------------------------------------

def test_attractive_dense_oracle(bh):
    rng = np.random.default_rng(13)
    n = 300
    a = np.triu(rng.random((n, n)) < 0.05, 1)
    mask = a | a.T
    w = np.triu(rng.random((n, n)), 1)
    w = (w + w.T) * mask
    w /= w.sum()
    rows, cols = np.nonzero(mask)
    ro = np.concatenate([[0], np.cumsum(mask.sum(axis=1))]).astype(np.int64)
    p = bh.from_csr(ro, cols.astype(np.int32), w[rows, cols])
    y = rng.standard_normal((n, 2))
    buf = bh.GradientBuffers.allocate(n, np.float64)
    bh.attractive(p, y, buf)
    diff = y[:, None, :] - y[None, :, :]
    q = 1.0 / (1.0 + (diff ** 2).sum(-1))
    ref = ((w * q)[:, :, None] * diff).sum(axis=1)
    np.testing.assert_allclose(buf.attr.cpu().numpy(), ref, rtol=1e-12,
                               atol=1e-17)


# --- the update (test_optimizer.py:53-141, 256-266) -------------------------

def _pair(bh, v=0.5):
    return bh.from_csr(np.array([0, 1, 2]), np.array([1, 0]), np.array([v, v]))


def _cfg(bh, **kw):
    base = dict(n_iter=10, exaggeration_iters=0, perplexity=2.0,
                precision="f64")
    base.update(kw)
    return bh.TsneConfig(**base)


def _emb(bh, y, v=None):
    return bh.embedding_from(np.asarray(y, np.float64),
                             v=None if v is None else np.asarray(v, np.float64))


def test_symmetric_pair_is_pure_momentum_decay(bh):
    y = [[-0.5, 0.0], [0.5, 0.0]]
    v = [[0.01, 0.005], [-0.02, 0.005]]
    e = _emb(bh, y, v)
    cfg = _cfg(bh, theta=0.0)
    bh.gradient_step(e, _pair(bh), cfg)
    expect = np.array(y) + cfg.momentum_early * np.array(v)
    expect -= expect.mean(axis=0)
    np.testing.assert_allclose(e.y.cpu().numpy(), expect, atol=1e-12)


def test_two_point_hand_trace(bh):
    y = np.array([[-1.0, 0.0], [1.0, 0.0]])
    p01 = 0.3
    k = 1.0 / (1.0 + 4.0)
    attr0 = p01 * k * (y[0] - y[1])
    rep0 = k * k * (y[0] - y[1])
    grad0 = 4.0 * (attr0 - rep0 / (2.0 * k))
    v0 = -200.0 * 1.2 * grad0  # first step: sign flip -> gain 1.2
    y0n, y1n = y[0] + v0, y[1] - v0
    mean = 0.5 * (y0n + y1n)
    e = _emb(bh, y)
    bh.gradient_step(e, _pair(bh, p01), _cfg(bh))
    got = e.y.cpu().numpy()
    np.testing.assert_allclose(got[0], y0n - mean, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(got[1], y1n - mean, rtol=1e-12, atol=1e-12)
    assert e.iteration == 1


def test_recentred_every_step(bh):
    n = 64
    idx = np.arange(n)
    cols = np.stack([(idx - 1) % n, (idx + 1) % n], axis=1)
    cols.sort(axis=1)
    p = bh.from_csr(np.arange(0, 2 * n + 1, 2), cols.ravel(),
                    np.full(2 * n, 1 / 128.0))
    e = bh.init_embedding(n, seed=5, dtype=np.float64)
    for _ in range(5):
        bh.gradient_step(e, p, _cfg(bh))
        m = e.y.cpu().numpy().mean(axis=0)
        assert abs(m[0]) <= 1e-12 and abs(m[1]) <= 1e-12


def test_gain_rule_and_floor(bh):
    e = _emb(bh, [[-1.0, 0.0], [1.0, 0.0]])
    bh.gradient_step(e, _pair(bh, 0.3), _cfg(bh))
    g = e.g.cpu().numpy()
    np.testing.assert_allclose(g[:, 0], [1.2, 1.2])  # sign flip: +0.2
    np.testing.assert_allclose(g[:, 1], [0.8, 0.8])  # sign(0) == sign(0): x0.8
    cfg = _cfg(bh, n_iter=50)
    for _ in range(30):
        bh.gradient_step(e, _pair(bh, 0.3), cfg)
    assert (e.g.cpu().numpy()[:, 1] >= cfg.min_gain).all()


@pytest.mark.parametrize("iteration,momentum", [(249, 0.5), (250, 0.8)])
def test_momentum_switch_f64(bh, iteration, momentum):
    e = _emb(bh, [[-0.5, 0.0], [0.5, 0.0]], [[0.02, 0.0], [-0.01, 0.0]])
    e.iteration = iteration
    v0 = e.v.cpu().numpy()[:, 0].copy()
    bh.gradient_step(e, _pair(bh), _cfg(bh, n_iter=300))
    np.testing.assert_allclose(e.v.cpu().numpy()[:, 0], momentum * v0, atol=1e-12)


# --- full runs on the digits set (test_acceptance.py:55-80, 292-300) --------

@pytest.fixture(scope="module")
def digits():
    sklearn = pytest.importorskip("sklearn.datasets")
    return sklearn.load_digits().data.astype(np.float64)


def test_digit_kl_band_and_trend(bh, digits):
    kls, hist = [], []
    for seed in range(3):
        _, timings, kl = bh.run(digits, bh.TsneConfig(seed=seed, kl_every=250,
                                                      precision="f64"))
        kls.append(kl)
        hist.append(dict(timings.kl_history))
    med = float(np.median(kls))
    assert 0.70 <= med <= 1.00, kls
    meds = [float(np.median([h[it] for h in hist])) for it in (250, 500, 1000)]
    assert meds[0] >= meds[1] >= meds[2], meds


def test_digit_precision_parity(bh, digits):
    kls = {}
    for precision in ("f64", "f32"):
        _, _, kls[precision] = bh.run(digits, bh.TsneConfig(seed=4,
                                                            precision=precision))
    assert abs(kls["f32"] - kls["f64"]) <= 0.02, kls
    assert math.isfinite(kls["f32"])
