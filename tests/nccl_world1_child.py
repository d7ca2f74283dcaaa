"""Child of tests/test_gpu_multirank.py::test_nccl_collectives_in_graphs (a
one-rank NCCL process group) and ::test_nccl_multi_gpu_bitwise (one rank per
GPU, boxes with >= 2 GPUs): the sharded engine with its collectives captured
in the iteration's CUDA graph, compared bitwise with the unsharded engine on
every rank.  Rank 0 prints one JSON line."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def main():
    import torch
    import torch.distributed as dist

    import paper_2212_11506_b200 as bh
    from paper_2212_11506_b200.dist import Shard
    from test_gpu_multirank import clustered_problem

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    dist.init_process_group("nccl", rank=rank, world_size=world)
    p, y0 = clustered_problem(bh)
    cfg = bh.TsneConfig(n_iter=130, exaggeration_iters=40, graph_chunk=10,
                        relabel_every=50)
    e1 = bh.embedding_from(y0)
    bh.Engine(p, e1, cfg).run(130)
    e2 = bh.embedding_from(y0)
    eng = bh.Engine(p, e2, cfg, shard=Shard(rank, world))
    eng.run(130)
    torch.cuda.synchronize()
    ok = [bool(eng.graphs_ok),
          bool(np.array_equal(e1.y.cpu().numpy(), e2.y.cpu().numpy())),
          bool(np.isfinite(e2.y.cpu().numpy()).all())]
    # every rank must agree (the full result is on every rank)
    flags = torch.tensor(ok, dtype=torch.int32, device="cuda")
    dist.all_reduce(flags, op=dist.ReduceOp.MIN)
    out = dict(zip(("graphs_ok", "equal", "finite"),
                   (bool(v) for v in flags.cpu().tolist())))
    dist.destroy_process_group()
    if rank == 0:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
