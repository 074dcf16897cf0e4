"""World-size-2 gloo test of the instance-sharded multi-GPU path (run on CPU): disjoint shards,
per-rank seeded weak-scaling batches, max-over-ranks time and sum-over-ranks work."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp

from paper_2509_01416_b200.distributed import rank_seed, shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as dist
    from paper_2509_01416_b200 import workloads as W
    from paper_2509_01416_b200.distributed import reduce_max, reduce_sum
    from tests import oracle_lib as O
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = W.config2(batch=3, n_cells=200, seed=rank_seed(rank))
    r = O.source_iteration(p.length, p.n_cells, 16, p.sigma_t, p.sigma_s0, p.source, O.make_config(1e-8), n_threads=1)
    upd = int(r["iterations"].astype(np.int64).sum()) * p.n_cells * 16
    t_local = 0.1 * (rank + 1)
    q.put((rank, upd, reduce_sum(upd), reduce_max(t_local), p.sigma_t[0, 0]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_reductions():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    total = sum(r[1] for r in res)
    assert all(r[2] == total for r in res)            # sum over ranks
    assert all(abs(r[3] - 0.2) < 1e-15 for r in res)  # max over ranks
    assert res[0][4] != res[1][4]                     # different per-rank instance batches


def test_shard_partition():
    for n, w in [(2048, 8), (10, 3), (5, 8)]:
        parts = [shard(n, r, w) for r in range(w)]
        assert parts[0][0] == 0 and parts[-1][1] == n
        assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))
