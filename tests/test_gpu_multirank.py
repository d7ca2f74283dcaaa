"""The multi-GPU engine (dist.Shard) at world sizes 2 and 4 on ONE GPU.

NCCL cannot place two ranks on one device, so the ranks run as threads of
this process with dist.LocalGroup collectives (stream-ordered copies behind
a rendezvous); everything else -- the partition kernel, the slot-range
force launch, the Z partial all-reduce, the sharded update, the packed Y
all-gather and unpack, the mean / bounds pass over the gathered Y, the
state gather of every relabel -- is the product code path.  The trajectory
must equal the single-GPU engine's bit for bit (the property that makes the
result independent of the GPU count), and the device partition must equal
its host mirror (dist.balanced_cuts).
"""

import numpy as np
import pytest

from conftest import golden

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bh():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2212_11506_b200 as m
    return m


def clustered_problem(bh, n=20_000, k=30, seed=3):
    """A clustered 2-D start with a kNN-like random P (symmetric CSR)."""
    rng = np.random.default_rng(seed)
    centres = rng.uniform(-20, 20, (12, 2))
    y0 = (centres[rng.integers(0, 12, n)]
          + rng.standard_normal((n, 2))).astype(np.float32) * 1e-3
    rows = np.repeat(np.arange(n), k)
    cols = (rows + rng.integers(1, 2000, n * k)) % n  # local-ish neighbours
    a = np.concatenate([rows, cols])
    b = np.concatenate([cols, rows])
    key = np.unique(a.astype(np.int64) * n + b)
    r, c = key // n, key % n
    v = rng.uniform(0.5, 1.5, key.shape[0])
    v = (v / v.sum()).astype(np.float32)
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(r, minlength=n), out=rp[1:])
    return bh.from_csr(rp, c.astype(np.int32), v), y0


def run_single(bh, p, y0, cfg, n_iter):
    e = bh.embedding_from(y0)
    bh.Engine(p, e, cfg).run(n_iter)
    return e.y.cpu().numpy(), e


def run_sharded(bh, p, y0, cfg, n_iter, world):
    from paper_2212_11506_b200.dist import run_local
    p.padded()  # build the shared padded CSR once, before the threads
    embs = [bh.embedding_from(y0) for _ in range(world)]

    def make(shard):
        return bh.Engine(p, embs[shard.rank], cfg, shard=shard)

    engines = run_local(world, make, n_iter)
    return [e.y.cpu().numpy() for e in embs], engines


@pytest.mark.parametrize("world", [2, 4])
def test_sharded_engine_bitwise_equals_single_gpu(bh, world):
    p, y0 = clustered_problem(bh)
    cfg = bh.TsneConfig(n_iter=130, exaggeration_iters=40, graph_chunk=10,
                        relabel_every=50)
    ref, _ = run_single(bh, p, y0, cfg, 130)
    ys, engines = run_sharded(bh, p, y0, cfg, 130, world)
    shares = [eng.share() for eng in engines]
    # the shares tile [0, n) and are not all equal (cost-balanced)
    assert shares[0][0] == 0 and shares[-1][1] == p.n
    assert all(a[1] == b[0] for a, b in zip(shares, shares[1:]))
    for y in ys:
        np.testing.assert_array_equal(y, ref)
    # velocity / gains gathered back at the end of the run equal too
    assert np.isfinite(ref).all()


def test_sharded_engine_f64_bitwise(bh):
    g = golden("affinity450f64")
    p = bh.from_csr(g["row_offsets"], g["col_indices"], g["values"])
    y0 = np.column_stack([g["y0_init"], g["y1_init"]])
    cfg = bh.TsneConfig(n_iter=60, exaggeration_iters=20, graph_chunk=10,
                        precision="f64", relabel_every=25)
    e1 = bh.embedding_from(y0)
    bh.Engine(p, e1, cfg).run(60)
    ys, _ = run_sharded(bh, p, y0, cfg, 60, 2)
    np.testing.assert_array_equal(ys[0], e1.y.cpu().numpy())
    np.testing.assert_array_equal(ys[1], e1.y.cpu().numpy())


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_device_partition_equals_host_mirror(bh, world):
    from paper_2212_11506_b200 import _lib
    from paper_2212_11506_b200._lib import call, ptr, stream
    from paper_2212_11506_b200.dist import W_POINT, balanced_cuts, share_cap
    rng = np.random.default_rng(world)
    for n in (100, 1000, 77_777):
        lens = rng.integers(4, 300, n) // 4 * 4 + 4
        lens[rng.integers(0, n, max(1, n // 40))] = 1204
        rp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        cap = share_cap(n, world)
        dev = _lib.device()
        rpt = torch.from_numpy(rp).to(dev)
        cuts = torch.zeros(world + 1, dtype=torch.int64, device=dev)
        parts = torch.zeros((world, 4), dtype=torch.int64, device=dev)
        call("bh_partition", ptr(rpt), n, world, W_POINT, 0.35, cap,
             ptr(cuts), ptr(parts), stream())
        host = balanced_cuts(rp, n, world, cap=cap)
        np.testing.assert_array_equal(cuts.cpu().numpy(), host)
        pt = parts.cpu().numpy()
        np.testing.assert_array_equal(pt[:, 0], host[:-1])
        np.testing.assert_array_equal(pt[:, 1], host[1:])
        np.testing.assert_array_equal(
            pt[:, 2], host[:-1] + np.floor(0.35 * np.diff(host)).astype(np.int64))


def test_nccl_collectives_in_graphs(bh):
    """The product transport: a one-rank NCCL group (two ranks cannot share
    a GPU), so the Z all-reduce and the Y all-gather run through
    ProcessGroupNCCL and are captured in the iteration's CUDA graph; the
    trajectory equals the unsharded engine's bitwise."""
    import json
    import os
    import socket
    import subprocess
    import sys
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
               RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
    child = os.path.join(os.path.dirname(os.path.abspath(__file__)),
                         "nccl_world1_child.py")
    r = subprocess.run([sys.executable, child], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out == {"graphs_ok": True, "equal": True, "finite": True}, (out, r.stderr[-2000:])


def test_nccl_multi_gpu_bitwise(bh):
    """One rank per GPU over NCCL (torchrun), world 2 (and 4 when the box
    has them): the sharded engine's trajectory equals the single-GPU one
    bitwise on every rank.  Needs >= 2 GPUs (skipped on one-GPU boxes, where
    dist.LocalGroup covers world 2 / 4 above)."""
    import json
    import os
    import socket
    import subprocess
    import sys

    import pytest
    import torch
    ngpu = torch.cuda.device_count()
    if ngpu < 2:
        pytest.skip("needs >= 2 GPUs")
    child = os.path.join(os.path.dirname(os.path.abspath(__file__)),
                         "nccl_world1_child.py")
    for world in [w for w in (2, 4) if w <= ngpu]:
        with socket.socket() as s:
            s.bind(("127.0.0.1", 0))
            port = s.getsockname()[1]
        r = subprocess.run(
            [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
             f"--nproc-per-node={world}", "--master-addr", "127.0.0.1",
             "--master-port", str(port), child],
            capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-3000:]
        line = [l for l in r.stdout.splitlines() if l.startswith("{")][-1]
        out = json.loads(line)
        assert out["equal"] and out["finite"], (world, out, r.stderr[-2000:])
