"""BHTM / CSV I/O (byte format of the reference io.py:1-30) on CPU, and the
bhtsne-compatible CLI on the GPU."""

import json
import struct

import numpy as np
import pytest

from paper_2212_11506_b200 import io


def test_bhtm_bytes_match_the_reference_layout(tmp_path):
    a = np.array([[1.5, -2.0], [3.25, 4.0]], np.float32)
    p = tmp_path / "m.bin"
    io.save_matrix(a, p)
    expect = b"BHTM" + struct.pack("<BQQ", 1, 2, 2) + a.astype("<f4").tobytes()
    assert p.read_bytes() == expect
    np.testing.assert_array_equal(io.load_matrix(p).data, a)
    b = a.astype(np.float64)
    io.save_matrix(b, p)
    assert p.read_bytes()[4] == 0
    np.testing.assert_array_equal(io.load_matrix(p, precision="f64").data, b)


def test_labels_and_package_exports(tmp_path):
    # io.py:120-128: one class id per non-empty line, first CSV field
    p = tmp_path / "labels.txt"
    p.write_text("3\n\n1.0,extra\n 7 \n")
    np.testing.assert_array_equal(io.load_labels(p), [3, 1, 7])
    assert io.load_labels(p).dtype == np.int64
    p.write_text("2\nnot-a-label\n")
    with pytest.raises(ValueError, match="labels file"):
        io.load_labels(p)
    import paper_2212_11506_b200 as pkg
    for name in ("InputMatrix", "load_matrix", "save_matrix", "load_labels"):
        assert getattr(pkg, name) is getattr(io, name) and name in pkg.__all__


def test_csv_round_trip_and_errors(tmp_path):
    a = np.random.default_rng(0).standard_normal((5, 3))
    p = tmp_path / "m.csv"
    io.save_matrix(a, p)
    np.testing.assert_array_equal(io.load_matrix(p, precision="f64").data, a)
    (tmp_path / "bad.csv").write_text("1,2\n3\n")
    with pytest.raises(ValueError, match="row 2 has 1 columns"):
        io.load_matrix(tmp_path / "bad.csv")
    (tmp_path / "nan.csv").write_text("1,2\n3,nan\n")
    with pytest.raises(ValueError, match="non-finite value at row 1, column 1"):
        io.load_matrix(tmp_path / "nan.csv")
    (tmp_path / "t.bin").write_bytes(b"BHTM" + struct.pack("<BQQ", 1, 4, 2))
    with pytest.raises(ValueError, match="truncated payload"):
        io.load_matrix(tmp_path / "t.bin")


def test_cli_parser_matches_reference_flags():
    from paper_2212_11506_b200.cli import build_parser
    p = build_parser()
    a = p.parse_args(["embed", "--input", "x.bin", "--out", "y.bin",
                      "--perplexity", "20", "--theta", "0.4", "--iters", "500",
                      "--learning-rate", "150", "--exaggeration", "8",
                      "--exaggeration-iters", "100", "--seed", "3",
                      "--threads", "4", "--precision", "f32", "--kl-every", "50"])
    assert (a.perplexity, a.theta, a.iters, a.exaggeration_iters) == (20, 0.4, 500, 100)


@pytest.mark.gpu
def test_cli_embed_writes_embedding_manifest_timings(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2212_11506_b200.cli import main
    from paper_2212_11506_b200.workloads import c0
    x = c0()[:600]
    inp = tmp_path / "x.bin"
    io.save_matrix(x, inp)
    out = tmp_path / "y.bin"
    rc = main(["embed", "--input", str(inp), "--out", str(out), "--iters", "300",
               "--exaggeration-iters", "100", "--perplexity", "20"])
    assert rc == 0
    y = io.load_matrix(out, precision="f64").data
    assert y.shape == (600, 2) and np.isfinite(y).all()
    m = json.loads((tmp_path / "y.bin.manifest.json").read_text())
    assert m["kl"] > 0 and m["config"]["n_iter"] == 300
    t = json.loads((tmp_path / "y.bin.timings.json").read_text())
    assert t["tree"]["calls"] == 300
    # reproducible from the manifest, bit for bit
    out2 = tmp_path / "y2.bin"
    assert main(["embed", "--input", str(inp), "--out", str(out2),
                 "--from-manifest", str(tmp_path / "y.bin.manifest.json")]) == 0
    assert out2.read_bytes() == out.read_bytes()
