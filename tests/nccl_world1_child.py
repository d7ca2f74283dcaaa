"""Child of tests/test_gpu_multirank.py::test_nccl_collectives_in_graphs: a
one-rank NCCL process group, the sharded engine with its collectives
captured in the iteration's CUDA graph, compared bitwise with the unsharded
engine.  Prints one JSON line."""
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

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1)
    p, y0 = clustered_problem(bh)
    cfg = bh.TsneConfig(n_iter=130, exaggeration_iters=40, graph_chunk=10,
                        relabel_every=50)
    e1 = bh.embedding_from(y0)
    bh.Engine(p, e1, cfg).run(130)
    e2 = bh.embedding_from(y0)
    eng = bh.Engine(p, e2, cfg, shard=Shard(0, 1))
    eng.run(130)
    torch.cuda.synchronize()
    out = {"graphs_ok": bool(eng.graphs_ok),
           "equal": bool(np.array_equal(e1.y.cpu().numpy(), e2.y.cpu().numpy())),
           "finite": bool(np.isfinite(e2.y.cpu().numpy()).all())}
    dist.destroy_process_group()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
