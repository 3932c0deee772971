"""Multi-process host logic of the N>1 path on CPU (gloo, world_size 2): sharding and the
single all-gather of results (paper_2312_06123_b200/dist.py).  The kernels themselves need
the GPU; here each rank's "results" are a known function of the global query index."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2312_06123_b200.dist import gather_results, shard


def test_shard_covers_exactly():
    for k in (0, 1, 7, 100, 10_001):
        for w in (1, 2, 3, 8):
            ranges = [shard(k, r, w) for r in range(w)]
            assert ranges[0][0] == 0 and ranges[-1][1] == k
            assert all(ranges[i][1] == ranges[i + 1][0] for i in range(w - 1))
            sizes = [hi - lo for lo, hi in ranges]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, k, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = shard(k, rank, world)
    local = torch.arange(lo, hi, dtype=torch.float64) * 0.5 + 1.0   # stand-in for r'(q)
    full = gather_results(local, k)
    q.put((rank, full.tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("k", [10, 11])
def test_gather_world2_gloo(k):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, k, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [i * 0.5 + 1.0 for i in range(k)]
    assert res[0] == want and res[1] == want
