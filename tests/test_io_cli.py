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


# --- the reference's CLI tests (pkg/tests/test_cli.py), restated -------------

@pytest.fixture
def cli(tmp_path):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2212_11506_b200.cli import main
    rng = np.random.default_rng(11)
    centres = np.array([[0.0, 0.0, 0.0], [8.0, 8.0, 8.0]])
    pts = np.vstack([c + rng.standard_normal((30, 3)) for c in centres])
    data = tmp_path / "data.csv"
    io.save_matrix(pts, data, format="csv")

    def embed_args(out, **extra):
        args = ["embed", "--input", str(data), "--out", str(out),
                "--perplexity", "5", "--iters", "50",
                "--exaggeration-iters", "20", "--seed", "1"]
        for key, val in extra.items():
            args += [f"--{key.replace('_', '-')}", str(val)]
        return args
    return main, data, embed_args


@pytest.mark.gpu
def test_cli_embed_outputs_and_exit_codes(cli, tmp_path, capsys):
    from paper_2212_11506_b200.optimizer import STAGES
    main, data, embed_args = cli
    out = tmp_path / "emb.csv"
    assert main(embed_args(out)) == 0
    emb = io.load_matrix(out, format="csv")
    assert (emb.n_points, emb.n_dims) == (60, 2)
    m = json.loads((tmp_path / "emb.csv.manifest.json").read_text())
    assert np.isfinite(m["kl"]) and m["seed"] == 1 and m["input"]["sha256"]
    t = json.loads((tmp_path / "emb.csv.timings.json").read_text())
    assert set(t) == set(STAGES)            # exactly the reference's stages
    assert "forces" in m["engine_timings"]
    # usage errors exit 2 with the reason, run-time errors return 1
    with pytest.raises(SystemExit) as exc:
        main(embed_args(tmp_path / "e.csv", perplexity="0.5"))
    assert exc.value.code == 2
    err = capsys.readouterr().err
    assert "perplexity" in err and "> 1" in err
    rc = main(["embed", "--input", str(tmp_path / "nope.csv"),
               "--out", str(tmp_path / "e.csv")])
    assert rc == 1 and "error" in capsys.readouterr().err
    # --threads is accepted and changes nothing (test_cli.py:59-65)
    outs = []
    for threads in (1, 8):
        o = tmp_path / f"emb{threads}.bin"
        assert main(embed_args(o, threads=threads)) == 0
        outs.append(o.read_bytes())
    assert outs[0] == outs[1]


@pytest.mark.gpu
def test_cli_profile_table_and_json(cli, tmp_path, capsys):
    from paper_2212_11506_b200.optimizer import STAGES
    main, data, _ = cli
    tj = tmp_path / "timings.json"
    assert main(["profile", "--input", str(data), "--perplexity", "5",
                 "--iters", "30", "--exaggeration-iters", "10",
                 "--timings-out", str(tj)]) == 0
    out = capsys.readouterr().out
    lines = [ln for ln in out.splitlines() if ln and not ln.startswith("wall")]
    body = [ln for ln in lines[1:] if not ln.startswith("total")]
    assert [ln.split()[0] for ln in body] == list(STAGES)
    pcts = [float(ln.split()[-1].rstrip("%")) for ln in body]
    assert abs(sum(pcts) - 100.0) <= 0.5
    report = json.loads(tj.read_text())
    assert set(report) == set(STAGES)
    for s in STAGES:
        assert report[s]["total_s"] >= 0
    # separate, non-overlapping kernels: every stage ran every iteration
    for s in ("tree", "summarize", "attractive", "repulsive", "update"):
        assert report[s]["calls"] == 30 and report[s]["total_s"] > 0


@pytest.mark.gpu
def test_cli_kl_matches_manifest_and_errors(cli, tmp_path, capsys):
    main, data, embed_args = cli
    out = tmp_path / "emb.bin"
    assert main(embed_args(out)) == 0
    m = json.loads((tmp_path / "emb.bin.manifest.json").read_text())
    capsys.readouterr()
    jout = tmp_path / "kl.json"
    printed = []
    for _ in range(2):
        assert main(["kl", "--input", str(data), "--embedding", str(out),
                     "--perplexity", "5", "--json-out", str(jout)]) == 0
        printed.append(capsys.readouterr().out)
    assert printed[0] == printed[1]                     # deterministic
    assert f"kl={m['kl']:.6f}" in printed[0]
    assert abs(json.loads(jout.read_text())["kl"] - m["kl"]) <= 1e-9
    short = tmp_path / "short.csv"
    io.save_matrix(np.random.default_rng(0).standard_normal((10, 2)), short,
                   format="csv")
    rc = main(["kl", "--input", str(data), "--embedding", str(short),
               "--perplexity", "5"])
    err = capsys.readouterr().err
    assert rc == 1 and "10" in err and "60" in err
