"""GPU parity at the benchmark's full size (C3: N = 1.3M points) through
size-independent properties: tree topology bit-exact against
the C oracle, the gradient against the oracle's to the north-star 1e-4
rel-L2, antisymmetry of the attraction, f32/f64 agreement, and bitwise
determinism of the graph-captured engine.  The 2-D state is a heavy-tailed
cluster mixture at the scale of a late C3 embedding; P is a random symmetric
K = 30 graph (the kNN is not part of the path).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

N = 1_300_000


@pytest.fixture(scope="module")
def bh():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2212_11506_b200 as m
    return m


@pytest.fixture(scope="module")
def state(bh):
    from paper_2212_11506_b200.affinity import PerplexityResult
    from paper_2212_11506_b200.workloads import c4_directed, c4_points
    y = c4_points(seed=3, n=N, k=40) * np.float32(0.5)
    idx, cond = c4_directed(seed=3, n=N, k=30)
    g = bh.NeighborGraph(idx.astype(np.int64), np.ones(idx.shape, np.float32))
    dev = torch.device("cuda")
    pr = PerplexityResult(betas=torch.ones(N, dtype=torch.float64, device=dev),
                          conditional=torch.from_numpy(cond).to(dev))
    p = bh.symmetrize(pr, g)
    return y, p


def test_fullsize_tree_bit_exact_vs_oracle(bh, oracle, state):
    y, _ = state
    c, r = bh.compute_bounds(y)
    assert (c, r) == oracle.compute_bounds(y)
    mc = bh.morton_codes(y, c, r)
    codes, order, sc = oracle.morton_codes(y, c, r, 32)
    np.testing.assert_array_equal(mc.codes_u64(), codes)
    np.testing.assert_array_equal(mc.order.cpu().numpy(), order)
    t = bh.summarize(bh.build_tree(mc, y))
    ot = oracle.tree_from_sorted(sc, order, y, c, r, 32)
    out = t.to_reference()
    for f in ("level_offsets", "start", "end", "children", "is_leaf", "mass",
              "com"):
        np.testing.assert_array_equal(out[f], getattr(ot, f), err_msg=f)


def test_fullsize_gradient_vs_oracle(bh, oracle, state):
    y, p = state
    ro, co, va = p.to_reference()
    g0, g1, _, _, z = oracle.gradient(y, ro, co, va, 0.5, code_bits=32)
    ref = np.column_stack([g0, g1]).astype(np.float64)
    c, r = bh.compute_bounds(y)
    t = bh.summarize(bh.build_tree(bh.morton_codes(y, c, r), y))
    buf = bh.GradientBuffers.allocate(N)
    bh.attractive(p, y, buf)
    bh.repulsive_bh(t, y, 0.5, buf)
    assert buf.z == pytest.approx(z, rel=1e-6)
    zf = np.float32(buf.z)
    got = 4.0 * (buf.attr.cpu().numpy().astype(np.float64)
                 - buf.rep.cpu().numpy().astype(np.float64) / zf)
    rel = np.linalg.norm(got - ref) / np.linalg.norm(ref)
    assert rel <= 1e-4, rel
    # attraction is antisymmetric over the symmetric P: sum_i attr_i = 0
    a = buf.attr.double()
    assert float(a.sum(0).norm()) <= 1e-6 * float(a.norm(dim=1).sum())


def test_fullsize_f32_and_f64_agree(bh, state):
    y, p = state
    out = {}
    for dt in (np.float32, np.float64):
        yy = y.astype(dt)
        pp = bh.from_csr(*p.to_reference()[:2], p.to_reference()[2].astype(dt))
        c, r = bh.compute_bounds(yy)
        t = bh.summarize(bh.build_tree(bh.morton_codes(yy, c, r), yy))
        buf = bh.GradientBuffers.allocate(N, dt)
        bh.attractive(pp, yy, buf)
        bh.repulsive_bh(t, yy, 0.5, buf)
        out[dt] = (buf.attr.double().cpu().numpy(), buf.rep.double().cpu().numpy(),
                   buf.z)
    (a32, r32, z32), (a64, r64, z64) = out[np.float32], out[np.float64]
    assert np.linalg.norm(a32 - a64) / np.linalg.norm(a64) < 1e-5
    assert np.linalg.norm(r32 - r64) / np.linalg.norm(r64) < 1e-5
    assert z32 == pytest.approx(z64, rel=1e-6)


def test_fullsize_engine_is_deterministic(bh, state):
    y, p = state
    outs = []
    for _ in range(2):
        e = bh.embedding_from(y)
        eng = bh.Engine(p, e, bh.TsneConfig(n_iter=300, exaggeration_iters=0,
                                            graph_chunk=10, relabel_every=10))
        e.iteration = 260
        eng.set_iteration(260)
        eng.run(30)
        outs.append(e.y.cpu().numpy())
    np.testing.assert_array_equal(outs[0], outs[1])
    assert np.isfinite(outs[0]).all()
