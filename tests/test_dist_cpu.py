"""Multi-process host logic of the N>1 path on CPU (gloo, world_size 2): sharding and the
single all-gather of results (paper_2312_06123_b200/dist.py).  The kernels themselves need
the GPU; here each rank's "results" are a known function of the global query index."""
import os
import socket

import numpy as np
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


def test_partition_covers_and_balances():
    from paper_2312_06123_b200.dist import partition, predicted_cost
    import workloads as W
    g, pairs, _ = W.load_config("tiny", with_lambda=False)
    cost = predicted_cost(pairs, g.degrees(), 0.6, 0.1)
    assert (cost > 0).all()
    for world in (1, 2, 3, 8):
        parts = partition(cost, world)
        allidx = np.sort(np.concatenate(parts))
        assert np.array_equal(allidx, np.arange(len(pairs)))            # a partition
        assert all(np.all(np.diff(p) > 0) for p in parts)                 # ascending per rank
        loads = np.array([cost[p].sum() for p in parts])
        assert loads.max() <= loads.mean() + cost.max()                   # within one item of even
        again = partition(cost, world)                                    # deterministic
        assert all(np.array_equal(a, b) for a, b in zip(parts, again))


def test_partition_heavy_tail_beats_contiguous():
    from paper_2312_06123_b200.dist import partition, shard
    rng = np.random.default_rng(1)
    cost = rng.lognormal(0.0, 1.0, 10_000)         # heavy-tailed per-query work
    cost[:500] *= 5.0                              # a cluster of expensive queries up front
    world = 8
    lpt = max(cost[p].sum() for p in partition(cost, world)) / (cost.sum() / world)
    cont = max(cost[lo:hi].sum() for lo, hi in (shard(len(cost), r, world) for r in range(world))) / (cost.sum() / world)
    assert lpt < 1.03 and cont > 1.3


def test_predicted_cost_matches_eq6_ell():
    """The cost model's ell is Eq. 6 (the oracle's refined_ell) on every query."""
    import oracle
    import workloads as W
    from paper_2312_06123_b200.dist import predicted_cost
    g, pairs, _ = W.load_config("tiny", with_lambda=False)
    d = g.degrees()
    lam, eps = 0.6, 0.1
    c = predicted_cost(pairs, d, lam, eps, fixed=0.0)
    for (s, t), ci in zip(pairs[:40], c[:40]):
        ell = oracle.refined_ell(int(d[s]), int(d[t]), eps, lam)
        assert np.isclose(ci, ell ** 3 * (1 / d[s] + 1 / d[t]) ** 2)


def _worker_part(rank, world, port, k, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2312_06123_b200.dist import gather_partitioned, partition
    cost = (np.arange(k) % 7 + 1.0) ** 2
    parts = partition(cost, world)
    idx = parts[rank]
    local = torch.as_tensor(idx, dtype=torch.float64) * 0.25 - 3.0     # stand-in for r'(q)
    full = gather_partitioned(local, parts)
    q.put((rank, full.tolist()))
    dist.destroy_process_group()


@pytest.mark.parametrize("k", [9, 16])
def test_gather_partitioned_world2_gloo(k):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_part, args=(r, 2, port, k, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [i * 0.25 - 3.0 for i in range(k)]
    assert res[0] == want and res[1] == want
