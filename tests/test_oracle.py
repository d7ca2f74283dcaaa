"""Pin the CPU oracle against golden vectors of the unmodified reference.

The fixtures come from tests/golden/make_golden.py (reference run in the
build container); mode 64 is the shipped reference, mode 32 the depth-16
reference (MAX_DEPTH = 16, top-32-bit codes, SURVEY.md 8(c) ii).
"""

import numpy as np
import pytest

from conftest import TREE_CASES, golden

TREE_ARRAYS = ("level_offsets", "start", "end", "children", "is_leaf",
               "cell_center", "cell_radius", "mass", "com", "order", "ys0",
               "ys1")


@pytest.mark.parametrize("mode", [64, 32])
@pytest.mark.parametrize("case", TREE_CASES)
def test_tree_bit_exact(oracle, mode, case):
    g = golden(f"tree{mode}_{case}")
    y = g["y"]
    center, r_span = oracle.compute_bounds(y)
    assert center == tuple(g["center"]) and r_span == float(g["r_span"])
    codes, order, sc = oracle.morton_codes(y, center, r_span, code_bits=mode)
    ref_codes = g["codes"] if mode == 64 else g["codes"] >> np.uint64(32)
    np.testing.assert_array_equal(codes, ref_codes)
    np.testing.assert_array_equal(order, g["order"])
    t = oracle.tree_from_sorted(sc, order, y, center, r_span, mode)
    for f in TREE_ARRAYS:
        np.testing.assert_array_equal(getattr(t, f), g[f], err_msg=f)


@pytest.mark.parametrize("case", TREE_CASES)
def test_32bit_codes_are_top_half_of_reference(oracle, case):
    """the 16-bit-per-dim code with scale 2^15/r_span is
    bit-for-bit the top 32 bits of the reference's 64-bit code."""
    y = golden(f"tree64_{case}")["y"]
    c, r = oracle.compute_bounds(y)
    c64, _, _ = oracle.morton_codes(y, c, r, 64)
    c32, _, _ = oracle.morton_codes(y, c, r, 32)
    np.testing.assert_array_equal(c32, c64 >> np.uint64(32))


def test_golden_dump(oracle):
    g = golden("tree64_dump4")
    t = oracle.build_tree(g["y"], code_bits=64)
    assert oracle.tree_dump(t) == str(g["dump"])
    # test_quadtree.py:306-316 literal
    assert oracle.tree_dump(t).splitlines()[0] == "0 - 4 -0.125 -0.125"


@pytest.mark.parametrize("mode", [64, 32])
@pytest.mark.parametrize("case", ["gauss2000", "heavy3200", "coinc7", "two",
                                  "quad4"])
@pytest.mark.parametrize("theta", [0.0, 0.5, 0.8])
def test_repulsive_bh_matches_reference(oracle, mode, case, theta):
    g = golden(f"tree{mode}_{case}")
    y = g["y"]
    t = oracle.build_tree(y, code_bits=mode)
    r0, r1, zp, z = oracle.repulsive_bh(t, y, theta)
    tag = f"bh{int(theta * 10)}"
    # same f64 operation order as forces.py:85-131 -> bit-exact
    np.testing.assert_array_equal(r0, g[tag + "_rep0"])
    np.testing.assert_array_equal(r1, g[tag + "_rep1"])
    np.testing.assert_array_equal(zp, g[tag + "_zpart"])
    assert z == pytest.approx(float(g[tag + "_z"]), rel=1e-14)


@pytest.mark.parametrize("case", ["gauss2000", "heavy3200", "coinc7", "two"])
def test_repulsive_exact_matches_reference(oracle, case):
    g = golden(f"tree64_{case}")
    r0, r1, zp, z = oracle.repulsive_exact(g["y"])
    np.testing.assert_array_equal(r0, g["ex_rep0"])
    np.testing.assert_array_equal(r1, g["ex_rep1"])
    np.testing.assert_array_equal(zp, g["ex_zpart"])


def test_calibrate_and_symmetrize(oracle):
    g = golden("affinity450")
    idx, sqd = oracle.knn_exact(g["x"], 30)
    np.testing.assert_array_equal(idx, g["indices"])
    np.testing.assert_array_equal(sqd, g["sq_distances"])
    betas, cond = oracle.calibrate_perplexity(g["sq_distances"], 10.0)
    # same schedule and sequential sums as affinity.py:61-96; libm exp/log
    # may differ from numba's by an ulp
    np.testing.assert_allclose(betas, g["betas"], rtol=1e-12)
    np.testing.assert_allclose(cond, g["cond"], rtol=1e-12, atol=1e-300)
    ro, co, va = oracle.symmetrize(g["indices"], g["cond"], np.float32)
    np.testing.assert_array_equal(ro, g["row_offsets"])
    np.testing.assert_array_equal(co, g["col_indices"])
    np.testing.assert_array_equal(va, g["values"])
    np.testing.assert_array_equal(oracle.exaggerate(va, 12.0), g["values12"])


def test_attractive_and_kl(oracle):
    g = golden("affinity450")
    a0, a1 = oracle.attractive(g["row_offsets"], g["col_indices"], g["values"],
                               g["y"])
    np.testing.assert_array_equal(a0, g["attr0"])
    np.testing.assert_array_equal(a1, g["attr1"])
    a0, a1 = oracle.attractive(g["row_offsets"], g["col_indices"],
                               g["values12"], g["y"])
    np.testing.assert_array_equal(a0, g["attr12_0"])
    np.testing.assert_array_equal(a1, g["attr12_1"])
    kl = oracle.kl_divergence(g["row_offsets"], g["col_indices"], g["values"],
                              g["y"])
    assert kl == pytest.approx(float(g["kl"]), rel=1e-12)


def test_attractive_two_point_closed_form(oracle):
    g = golden("closed_forms")
    a0, a1 = oracle.attractive(np.array([0, 1, 2]), np.array([1, 0]),
                               np.array([0.5, 0.5], np.float32),
                               np.array([[0.0, 0.0], [1.0, 0.0]], np.float32))
    np.testing.assert_array_equal(np.column_stack([a0, a1]), g["attr_two"])
    np.testing.assert_array_equal(a0, [-0.25, 0.25])


def test_gradient_step_trajectory(oracle):
    """Eight reference gradient_step calls (f32 run mode), exaggerated then
    not, across the momentum switch; the oracle restates the update with
    numpy's float32 semantics (NEP 50)."""
    a = golden("affinity450")
    g = golden("trajectory450")
    s = oracle.State.init(450, 3)
    np.testing.assert_array_equal(s.y0, g["y0_init"])
    v12 = oracle.exaggerate(a["values"], 12.0)
    for it in range(8):
        if it == 4:
            s.iteration = 250
        vals = v12 if it < 4 else a["values"]
        oracle.gradient_step(s, a["row_offsets"], a["col_indices"], vals,
                             code_bits=64)
        # the mean is a f64 sum whose order differs from numpy's pairwise
        # sum; after the f32 cast it agrees to the last bit or one ulp
        np.testing.assert_allclose(s.y0, g[f"y0_{it}"], rtol=0, atol=1e-9)
        np.testing.assert_allclose(s.y1, g[f"y1_{it}"], rtol=0, atol=1e-9)
        np.testing.assert_array_equal(s.g0, g[f"g0_{it}"])
        np.testing.assert_allclose(s.v0, g[f"v0_{it}"], rtol=1e-6, atol=1e-12)


def test_c0_knn_matches_reference(oracle):
    from paper_2212_11506_b200.workloads import c0
    g = golden("c0_run")
    idx, _ = oracle.knn_exact(c0(), 90)
    np.testing.assert_array_equal(idx, g["indices"].astype(np.int64))


@pytest.mark.slow
def test_c0_full_run_kl(oracle):
    """C0 full 1000-iteration run: oracle KL within 1% of the reference."""
    from paper_2212_11506_b200.workloads import c0
    g = golden("c0_run")
    idx, sqd = oracle.knn_exact(c0(), 90)
    s, kl, _ = oracle.run(idx, sqd, n_iter=1000, code_bits=64)
    assert abs(kl - float(g["kl"])) / float(g["kl"]) < 0.01
