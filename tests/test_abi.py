"""CPU checks of the boundary: the sm_100a library builds, loads without a
GPU and exports every symbol include/bhtsne_b200.h declares; host-side
logic (config validation, estimator validation, struct layouts)."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "bhtsne_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"\b(bh_[a-z0-9_]+)\s*\(", src)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    from paper_2212_11506_b200 import _build, _lib
    _build.build()
    return _lib.load_symbols_only()


def test_library_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 25
    for name in names:
        assert hasattr(lib, name), name
    from paper_2212_11506_b200._lib import SIGNATURES
    assert set(SIGNATURES) == set(names)


def test_library_is_sm100a(lib):
    from paper_2212_11506_b200._lib import LIB_PATH
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                          LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_version_and_bounds(lib):
    assert lib.bh_abi_version() == 1
    assert lib.bh_tree_node_bound(1000, 32) == 1000 * 17 + 1
    assert lib.bh_tree_node_bound(10, 64) == 10 * 33 + 1
    assert lib.bh_sort_workspace_bytes(1 << 20, 32) > 8 * (1 << 20)


def test_struct_layouts_match_header():
    """Compile a tiny C program against the header and compare sizes /
    offsets with the ctypes/numpy views used by the host."""
    from paper_2212_11506_b200._lib import BOUNDS_DTYPE, SCHED_DTYPE, TreeStruct
    prog = r"""
    #include <stdio.h>
    #include <stddef.h>
    #include "bhtsne_b200.h"
    int main(void) {
      printf("%zu %zu %zu %zu %zu %zu\n", sizeof(bh_bounds_t), sizeof(bh_sched_t),
             sizeof(bh_tree_t), offsetof(bh_sched_t, z),
             offsetof(bh_tree_t, status), offsetof(bh_bounds_t, shift0));
      return 0;
    }"""
    tmp = os.path.join(REPO, "build")
    os.makedirs(tmp, exist_ok=True)
    c = os.path.join(tmp, "layout.c")
    exe = os.path.join(tmp, "layout")
    open(c, "w").write(prog)
    subprocess.run(["gcc", "-I", os.path.join(REPO, "include"), c, "-o", exe],
                   check=True)
    vals = [int(v) for v in subprocess.run([exe], capture_output=True,
                                           text=True).stdout.split()]
    assert vals[0] == BOUNDS_DTYPE.itemsize
    assert vals[1] == SCHED_DTYPE.itemsize
    assert vals[2] == ctypes.sizeof(TreeStruct)
    assert vals[3] == SCHED_DTYPE.fields["z"][1]
    assert vals[4] == TreeStruct.status.offset
    assert vals[5] == BOUNDS_DTYPE.fields["shift0"][1]


def test_no_oracle_in_product_package():
    pkg = os.path.join(REPO, "paper_2212_11506_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                src = open(os.path.join(root, f)).read()
                assert "oracle" not in src.replace("oracle/", "").lower() or \
                    f in ("__init__.py",), f"{f} mentions the oracle"


def test_product_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2212_11506_b200 as bh
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        bh.compute_bounds(np.zeros((4, 2), np.float32))


def test_config_validation_messages():
    from paper_2212_11506_b200 import TsneConfig
    with pytest.raises(ValueError, match="perplexity"):
        TsneConfig(perplexity=0.5).validate()
    with pytest.raises(ValueError, match="theta"):
        TsneConfig(theta=-1).validate()
    with pytest.raises(ValueError, match="learning rate"):
        TsneConfig(learning_rate=0).validate()
    with pytest.raises(ValueError, match="exaggeration phase"):
        TsneConfig(n_iter=100, exaggeration_iters=250).validate()
    with pytest.raises(ValueError, match="precision"):
        TsneConfig(precision="f16").validate()
    with pytest.raises(ValueError, match="code_bits"):
        TsneConfig(code_bits=48).validate()
    TsneConfig().validate()


def test_estimator_validation():
    from paper_2212_11506_b200 import BarnesHutTSNE
    with pytest.raises(ValueError, match="perplexity"):
        BarnesHutTSNE(perplexity=1.0)
    with pytest.raises(ValueError, match="nIter"):
        BarnesHutTSNE(n_iter=-3)
    est = BarnesHutTSNE()
    with pytest.raises(ValueError, match="at least 2 rows"):
        est.fit_transform(np.zeros((1, 3)))
    with pytest.raises(ValueError, match="non-finite value at row 1"):
        est.fit_transform(np.array([[0.0, 1.0], [np.nan, 2.0]]))


def test_morton_interleave_host_helper():
    from paper_2212_11506_b200 import morton_interleave
    assert morton_interleave(3, 7) == 47
    assert morton_interleave(0, 0) == 0


def test_partial_granularity_matches_header():
    """dist.ShardPlan aligns ranges to the traversal CTA's Z partial size,
    which the library static_asserts against the header macro."""
    import re
    from paper_2212_11506_b200.dist import POINTS_PER_PARTIAL
    with open(HEADER) as fh:
        m = re.search(r"#define BH_REP_POINTS_PER_PARTIAL (\d+)", fh.read())
    assert m and int(m.group(1)) == POINTS_PER_PARTIAL
