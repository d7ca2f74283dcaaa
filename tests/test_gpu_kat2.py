"""The rest of the reference's known-answer tests (pkg/tests: test_knn.py,
test_forces.py:116-149, test_quadtree.py:22-84, test_optimizer.py:28-47,
157-253), restated against the CUDA path through the public API -- the
cases tests/test_gpu_kat.py does not already hold: kNN edge cases, the exact
repulsion's symmetries, bounds and code edge cases, KL identities, config
validation and the run() bookkeeping.  float64 inputs run the `_f64` kernels
with the reference's tolerances.
"""

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
    return np.random.default_rng(4321)


def host(t):
    return t.detach().cpu().numpy()


# --- exact kNN (test_knn.py) ------------------------------------------------

def brute_force(data, k):
    """Dense distances, per-row lexsort on (distance, id): ties -> lower id."""
    n = data.shape[0]
    d2 = np.zeros((n, n))
    for c in range(data.shape[1]):          # column order, as knn.py:36-59
        diff = data[:, None, c] - data[None, :, c]
        d2 = d2 + diff * diff
    np.fill_diagonal(d2, np.inf)
    ids = np.arange(n)
    idx = np.stack([np.lexsort((ids, d2[i]))[:k] for i in range(n)])
    return idx, np.take_along_axis(d2, idx, axis=1)


def test_knn_collinear_and_ties(bh):
    g = bh.knn_exact(np.array([[0.0], [1.0], [10.0]]), 1)
    np.testing.assert_array_equal(host(g.indices)[:, 0], [1, 0, 1])
    np.testing.assert_array_equal(host(g.sq_distances)[:, 0], [1.0, 1.0, 81.0])
    # unit square: corners 1 and 2 tie for corner 0 -> the lower id first
    sq = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])
    g = bh.knn_exact(sq, 3)
    np.testing.assert_array_equal(host(g.indices)[0], [1, 2, 3])
    np.testing.assert_array_equal(host(g.indices)[3], [1, 2, 0])


def test_knn_k_equals_n_minus_1_is_a_permutation(bh, rng):
    g = bh.knn_exact(rng.standard_normal((20, 3)), 19)
    idx = host(g.indices)
    for i in range(20):
        assert set(idx[i]) == set(range(20)) - {i}


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_knn_matches_brute_force(bh, rng, dtype):
    data = rng.standard_normal((200, 5)).astype(dtype)
    g = bh.knn_exact(data, 15)
    idx, sqd = brute_force(data.astype(np.float64), 15)
    np.testing.assert_array_equal(host(g.indices), idx)
    assert host(g.sq_distances).dtype == dtype
    if dtype == np.float64:   # the same f64 column-order sums: bitwise
        np.testing.assert_array_equal(host(g.sq_distances), sqd)
    else:
        np.testing.assert_array_equal(host(g.sq_distances),
                                      sqd.astype(np.float32))


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("offset,scale", [(1e4, 1.0), (1e6, 1.0), (0.0, 1e-20),
                                          (0.0, 1e25)])
def test_knn_filter_is_only_a_filter(bh, rng, dtype, offset, scale):
    """The f32 dot-product filter (k_knn_tile) may only drop pairs it proves
    too far: data far from the origin (|x|^2 >> d^2, where its bound is
    weakest), tiny values (f32 underflow of the norms) and huge ones (f32
    overflow -> NaN bounds, every pair taken exactly) still give the
    brute-force graph bit for bit."""
    if dtype == np.float32 and scale > 1e18:
        pytest.skip("squared distances overflow float32 itself")
    n, d, k = 700, 20, 30
    data = ((rng.standard_normal((n, d)) + offset) * scale).astype(dtype)
    g = bh.knn_exact(data, k)
    idx, sqd = brute_force(data.astype(np.float64), k)
    np.testing.assert_array_equal(host(g.indices), idx)
    np.testing.assert_array_equal(host(g.sq_distances), sqd.astype(dtype))


def test_knn_rows_sorted_valid_and_bounding(bh, rng):
    data = rng.standard_normal((100, 4))
    k = 10
    g = bh.knn_exact(data, k)
    idx, sqd = host(g.indices), host(g.sq_distances)
    d2 = ((data[:, None, :] - data[None, :, :]) ** 2).sum(-1)
    for i in range(100):
        assert (np.diff(sqd[i]) >= 0).all()
        assert (sqd[i] >= 0).all() and np.isfinite(sqd[i]).all()
        assert i not in idx[i] and len(set(idx[i])) == k
        rest = np.setdiff1d(np.arange(100), np.r_[idx[i], i])
        assert sqd[i].max() <= d2[i, rest].min() + 1e-15


def test_knn_is_deterministic(bh, rng):
    # the reference's thread-count invariance (test_knn.py:78-89): repeated
    # launches give the same bytes
    data = rng.standard_normal((150, 6))
    a, b = bh.knn_exact(data, 12), bh.knn_exact(data, 12)
    assert torch.equal(a.indices, b.indices)
    assert torch.equal(a.sq_distances.view(torch.uint8),
                       b.sq_distances.view(torch.uint8))


def test_knn_k_out_of_range(bh, rng):
    x = rng.standard_normal((5, 2))
    for k in (0, 5):
        with pytest.raises(ValueError, match="k must be"):
            bh.knn_exact(x, k)


# --- exact repulsion (test_forces.py:116-149) --------------------------------

def test_exact_square_symmetry(bh):
    y = np.array([[1.0, 1.0], [-1.0, 1.0], [-1.0, -1.0], [1.0, -1.0]])
    buf = bh.GradientBuffers.allocate(4, np.float64)
    bh.repulsive_exact(y, buf)
    rep = host(buf.rep)
    for i in range(4):  # outward along the corner's diagonal
        np.testing.assert_allclose(rep[i] / np.abs(rep[i]).max(),
                                   y[i] / np.abs(y[i]).max(), rtol=1e-12)
    np.testing.assert_allclose(rep.sum(axis=0), [0.0, 0.0], atol=1e-12)


def test_exact_forces_sum_to_zero(bh, rng):
    y = rng.standard_normal((250, 2)) * 5
    buf = bh.GradientBuffers.allocate(250, np.float64)
    bh.repulsive_exact(y, buf)
    np.testing.assert_allclose(host(buf.rep).sum(axis=0), [0.0, 0.0],
                               atol=1e-10 * 250)


def test_exact_matches_cost_gradient(bh, rng):
    # F_rep_i / Z = sum_j q_ij^2 Z (y_i - y_j), straight from the cost
    n = 100
    y = rng.standard_normal((n, 2)) * 2
    diff = y[:, None, :] - y[None, :, :]
    kern = 1.0 / (1.0 + (diff ** 2).sum(-1))
    np.fill_diagonal(kern, 0.0)
    z = kern.sum()
    want = ((kern / z)[:, :, None] ** 2 * z * diff).sum(axis=1)
    buf = bh.GradientBuffers.allocate(n, np.float64)
    bh.repulsive_exact(y, buf)
    np.testing.assert_allclose(host(buf.rep) / buf.z, want, rtol=1e-10,
                               atol=1e-15)
    assert buf.z == pytest.approx(z, rel=1e-12)


# --- bounds and codes (test_quadtree.py:22-84) --------------------------------

def test_bounds_edge_cases(bh):
    center, r_span = bh.compute_bounds(np.array([[0.0, 0.0], [2.0, 2.0]]), 64)
    assert center == (1.0, 1.0) and r_span >= 1.0
    center, r_span = bh.compute_bounds(np.array([[3.0, 3.0], [3.0, 3.0]]), 64)
    assert center == (3.0, 3.0) and r_span > 0   # epsilon floor
    with pytest.raises(ValueError, match="non-finite"):
        bh.compute_bounds(np.array([[0.0, np.inf], [1.0, 1.0]]))
    with pytest.raises(ValueError, match="non-finite"):
        bh.compute_bounds(np.array([[np.nan, 0.0], [1.0, 1.0]]))


@pytest.mark.parametrize("spread", [1e-6, 1.0, 1e6])
@pytest.mark.parametrize("code_bits", [32, 64])
def test_scaled_coordinates_in_range_and_codes(bh, rng, spread, code_bits):
    y = rng.standard_normal((2000, 2)) * spread
    center, r_span = bh.compute_bounds(y, code_bits)
    half = code_bits // 2
    scale = 2.0 ** (half - 1) / r_span
    m = (y - (np.array(center) - r_span)) * scale
    assert (m >= 0).all() and (m < 2.0 ** half).all()
    mc = bh.morton_codes(y, center, r_span, code_bits)
    codes = host(mc.codes).astype(np.uint64 if code_bits == 64 else np.uint32)
    for i in range(0, 2000, 37):
        want = bh.morton_interleave(int(m[i, 0]), int(m[i, 1]))
        assert int(codes[i]) == want


def test_interleave_known_answers(bh, rng):
    assert bh.morton_interleave(3, 7) == 47      # 101111b
    assert bh.morton_interleave(0, 0) == 0
    assert bh.morton_interleave(2 ** 32 - 1, 0) == 0x5555555555555555
    assert bh.morton_interleave(0, 2 ** 32 - 1) == 0xAAAAAAAAAAAAAAAA
    # the device interleave against the per-bit definition on corner cells
    y = np.array([[-1.0, -1.0], [1.0, 1.0], [-1.0, 1.0], [1.0, -1.0],
                  [0.0, 0.0]])
    center, r_span = bh.compute_bounds(y, 64)
    codes = host(bh.morton_codes(y, center, r_span, 64).codes).astype(np.uint64)
    scale = 2.0 ** 31 / r_span
    for i in range(5):
        m0 = int((y[i, 0] - (center[0] - r_span)) * scale)
        m1 = int((y[i, 1] - (center[1] - r_span)) * scale)
        assert int(codes[i]) == bh.morton_interleave(m0, m1)


# --- init, KL, config, run (test_optimizer.py) --------------------------------

def test_init_deterministic_and_statistics(bh):
    a, b = bh.init_embedding(100, seed=42), bh.init_embedding(100, seed=42)
    assert torch.equal(a.y, b.y)
    assert not torch.equal(a.y, bh.init_embedding(100, seed=43).y)
    e = bh.init_embedding(10_000, seed=7, dtype=np.float64)
    y = host(e.y)
    for col in (y[:, 0], y[:, 1]):
        assert 0.9e-4 <= col.std() <= 1.1e-4
        assert abs(col.mean()) <= 3.0 * 1e-4 / np.sqrt(10_000)
    assert (host(e.g) == 1.0).all() and (host(e.v) == 0.0).all()
    assert e.iteration == 0
    assert bh.init_embedding(50, seed=1, dtype=np.float32).y.dtype == torch.float32
    # the same Philox stream as the reference: f32 is the rounded f64 draw
    e32 = bh.init_embedding(10_000, seed=7, dtype=np.float32)
    np.testing.assert_array_equal(host(e32.y), y.astype(np.float32))


def three_points(bh):
    y = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 5.0]])
    p = bh.from_csr(np.array([0, 1, 2, 2], np.int64),
                    np.array([1, 0], np.int64), np.array([0.5, 0.5]))
    return y, p


def test_kl_hand_trace_and_isometry(bh):
    y, p = three_points(bh)
    buf = bh.GradientBuffers.allocate(3, np.float64)
    bh.repulsive_exact(y, buf)
    q01 = (1.0 / (1.0 + 1.0)) / buf.z
    want = 2 * (0.5 * np.log(0.5 / q01))
    base = bh.kl_divergence(p, y)
    assert base == pytest.approx(want, rel=1e-12)
    a = 0.7
    rot = np.array([[np.cos(a), -np.sin(a)], [np.sin(a), np.cos(a)]])
    moved = y @ rot.T + np.array([3.0, -2.0])
    assert abs(bh.kl_divergence(p, moved) - base) <= 1e-10


def test_kl_exact_vs_bh_theta0_and_errors(bh, rng):
    y = rng.standard_normal((300, 2))
    g = bh.knn_exact(rng.standard_normal((300, 6)), 30)
    p = bh.symmetrize(bh.calibrate_perplexity(g, 10.0), g)
    exact = bh.kl_divergence(p, y, mode="exact")
    bh0 = bh.kl_divergence(p, y, mode="bh", theta=0.0)
    assert abs(exact - bh0) <= 1e-10 * abs(exact)
    y3, p3 = three_points(bh)
    with pytest.raises(ValueError, match="exaggeration"):
        bh.kl_divergence(bh.set_exaggeration(p3, 12.0), y3)
    with pytest.raises(ValueError, match="mode"):
        bh.kl_divergence(p3, y3, mode="approx")
    with pytest.raises(ValueError, match="points"):
        bh.kl_divergence(p3, np.zeros((4, 2)))


def test_config_validation(bh):
    C = bh.TsneConfig
    with pytest.raises(ValueError, match="perplexity"):
        C(perplexity=0.5).validate()
    with pytest.raises(ValueError, match="theta"):
        C(theta=-1).validate()
    with pytest.raises(ValueError, match="learning rate"):
        C(learning_rate=0).validate()
    with pytest.raises(ValueError, match="exaggeration phase"):
        C(n_iter=100, exaggeration_iters=250).validate()
    with pytest.raises(ValueError, match="precision"):
        C(precision="f16").validate()
    assert C().validate().perplexity == 30.0 and C().theta == 0.5


@pytest.mark.parametrize("precision", ["f32", "f64"])
def test_run_zero_iterations(bh, rng, precision):
    x = rng.standard_normal((40, 5))
    cfg = bh.TsneConfig(n_iter=0, exaggeration_iters=0, perplexity=5.0,
                        seed=9, precision=precision)
    e, timings, kl = bh.run(x, cfg)
    assert torch.equal(e.y, bh.init_embedding(40, 9, dtype=cfg.dtype).y)
    assert np.isfinite(kl) and kl > 0
    assert timings.calls("tree") == 0


def test_run_bookkeeping_and_kl_history(bh, rng):
    x = rng.standard_normal((120, 8))
    cfg = bh.TsneConfig(n_iter=60, exaggeration_iters=20, perplexity=8.0,
                        seed=2, threads=2)
    e, timings, kl = bh.run(x, cfg, profile=True)
    assert torch.isfinite(e.y).all() and np.isfinite(kl)
    for stage in bh.STAGES:
        assert stage in timings.per_call
    assert timings.calls("tree") == 60 and timings.calls("knn") == 1
    assert sum(timings.total(s) for s in bh.STAGES) <= timings.total_wall_s
    assert e.iteration == 60
    x = rng.standard_normal((60, 5))
    cfg = bh.TsneConfig(n_iter=40, exaggeration_iters=0, perplexity=6.0,
                        kl_every=20, seed=1)
    _, timings, _ = bh.run(x, cfg)
    assert [it for it, _ in timings.kl_history] == [20, 40]


def test_run_improves_kl(bh, rng):
    centers = rng.standard_normal((4, 6)) * 8
    x = np.vstack([c + rng.standard_normal((30, 6)) for c in centers])
    base = dict(perplexity=10.0, seed=3)
    _, _, kl0 = bh.run(x, bh.TsneConfig(n_iter=0, exaggeration_iters=0, **base))
    _, _, kl = bh.run(x, bh.TsneConfig(n_iter=300, exaggeration_iters=100,
                                       **base))
    assert kl < kl0
