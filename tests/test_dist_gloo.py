"""The N>1 host path on CPU: 2 gloo ranks (127.0.0.1) exercise the cross-rank
reduction used by bench.py (max of times, sum of work) and the disjoint request
sharding of weak scaling."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    from paper_2504_18154_b200.dist import reduce_max_sum, shard_requests
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mx, sm = reduce_max_sum([10.0 + rank, 100.0 * (rank + 1)])
    ids = list(shard_requests(10, rank, world))
    dist.barrier()
    q.put((rank, mx, sm, ids))
    dist.destroy_process_group()


def test_two_rank_reduction_and_sharding():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = dict((r, (mx, sm, ids)) for r, mx, sm, ids in (q.get(timeout=120) for _ in range(2)))
    for p in ps:
        p.join(timeout=60)
    for r in (0, 1):
        assert out[r][0] == [11.0, 200.0]        # max over ranks (times)
        assert out[r][1] == [21.0, 300.0]        # sum over ranks (work)
    assert sorted(out[0][2] + out[1][2]) == list(range(10)) and not set(out[0][2]) & set(out[1][2])
