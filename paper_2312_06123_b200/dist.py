"""Multi-GPU plumbing: one process per GPU, queries sharded, results all-gathered.

The graph (CSR) is replicated on every rank; queries are independent, so
each rank answers its own subset of the query list.  Every query keeps its GLOBAL index
(``er_opts.query_ids``; ``query_index_base`` for contiguous shards), which keys its RNG
streams (R10): no output bit depends on the number of GPUs or on which rank ran
a query.  The only collective is one all-gather of the fp64 results (torch.distributed;
NCCL over NVLink on the GPU box, gloo in the CPU tests).

Two shardings:
  ``shard``      contiguous balanced ranges (weak-scaling bench: each rank its own set);
  ``partition``  a deterministic cost-model split of ONE global query list (strong
                 scaling).  Per-query work is heavy-tailed (CV ~ 4-5 of walk
                 steps at config 1), so a random split of 10k queries over 8 ranks loses
                 ~20% to the slowest rank.  The predicted cost of (s, t) is Eq. 13's shape,
                 ell^3 (1/d_s + 1/d_t)^2 with ell from Eq. 6 (degrees and lambda only),
                 plus a per-query constant; queries are dealt to ranks in boustrophedon order
                 of decreasing cost (a vectorised approximation of LPT).  Every rank computes
                 the same partition from the full pair list: no collective is needed for it.
This module is host-side plumbing: it never computes an estimate.
"""
from __future__ import annotations

import numpy as np


def shard(k_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous balanced split of [0, k_total): rank r gets [lo, hi)."""
    if world < 1 or not (0 <= rank < world) or k_total < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(k_total, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def predicted_cost(pairs: np.ndarray, degrees: np.ndarray, lam: float, eps: float,
                   fixed: float = 1.0) -> np.ndarray:
    """Relative work of each query: ell^3 (1/d_s + 1/d_t)^2 + fixed, ell by Eq. 6
    (s = t costs nothing but the fixed part)."""
    p = np.asarray(pairs, dtype=np.int64).reshape(-1, 2)
    ds = degrees[p[:, 0]].astype(np.float64)
    dt = degrees[p[:, 1]].astype(np.float64)
    inv = 1.0 / ds + 1.0 / dt
    x = np.log((2.0 * inv) / (eps * (1.0 - lam))) / np.log(1.0 / lam) - 1.0
    ell = np.maximum(0.0, np.ceil(x))
    cost = ell ** 3 * inv ** 2 + fixed
    cost[p[:, 0] == p[:, 1]] = fixed
    return cost


def partition(cost: np.ndarray, world: int) -> list[np.ndarray]:
    """Deterministic split of queries 0..k-1 into `world` index lists (ascending within a
    rank) with near-equal total cost: sort by decreasing cost (stable), deal in
    boustrophedon order 0..W-1, W-1..0, ..."""
    if world < 1:
        raise ValueError("world must be >= 1")
    k = len(cost)
    order = np.argsort(-np.asarray(cost, dtype=np.float64), kind="stable")
    pos = np.arange(k)
    rnd, off = np.divmod(pos, world)
    rank_of = np.where(rnd % 2 == 0, off, world - 1 - off)
    owner = np.empty(k, dtype=np.int64)
    owner[order] = rank_of
    return [np.nonzero(owner == r)[0] for r in range(world)]


def gather_results(out_local, k_total: int, group=None):
    """All-gather every rank's fp64 results of a CONTIGUOUS ``shard`` into a [k_total]
    tensor in global order.

    Shards may differ in length by one (``shard``); each rank pads to the largest
    shard, one ``all_gather_into_tensor`` moves k_total*8 bytes (plus padding), and
    the padding is dropped.
    """
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    sizes = [shard(k_total, r, world) for r in range(world)]
    mx = max(hi - lo for lo, hi in sizes)
    buf = torch.zeros(mx, dtype=out_local.dtype, device=out_local.device)
    buf[: out_local.numel()] = out_local
    allbuf = torch.empty(mx * world, dtype=out_local.dtype, device=out_local.device)
    dist.all_gather_into_tensor(allbuf, buf, group=group)
    parts = [allbuf[r * mx: r * mx + (hi - lo)] for r, (lo, hi) in enumerate(sizes)]
    return torch.cat(parts)


def gather_partitioned(out_local, parts: list[np.ndarray], group=None):
    """All-gather the results of a ``partition``: rank r holds out_local[j] = r'(parts[r][j]);
    returns the [k_total] tensor in global (input) order on every rank."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    assert len(parts) == world
    k_total = sum(len(p) for p in parts)
    mx = max(len(p) for p in parts)
    buf = torch.zeros(mx, dtype=out_local.dtype, device=out_local.device)
    buf[: out_local.numel()] = out_local
    allbuf = torch.empty(mx * world, dtype=out_local.dtype, device=out_local.device)
    dist.all_gather_into_tensor(allbuf, buf, group=group)
    full = torch.empty(k_total, dtype=out_local.dtype, device=out_local.device)
    for r, idx in enumerate(parts):
        if len(idx):
            full[torch.as_tensor(idx, device=out_local.device)] = allbuf[r * mx: r * mx + len(idx)]
    return full


def query_sharded(G, h, pairs: np.ndarray, eps: float, p_fail: float, degrees: np.ndarray, lam: float,
                  group=None, **kw):
    """Answer one global query list on all ranks of `group`: cost-model partition, each rank
    runs its part through the C ABI with global query ids, one all-gather.  Returns the
    results of all queries (input order) as a device tensor on every rank."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    parts = partition(predicted_cost(pairs, degrees, lam, eps), world)
    idx = parts[rank]
    dev = torch.device("cuda", torch.cuda.current_device())
    out = torch.zeros(len(idx), dtype=torch.float64, device=dev)
    if len(idx):
        sub = torch.from_numpy(np.ascontiguousarray(pairs[idx], dtype=np.int32)).to(dev)
        ids = torch.from_numpy(idx.astype(np.int64)).to(dev)
        G.er_query_batch_ex(h, sub, eps, p_fail, out=out, query_ids=ids, **kw)
    return gather_partitioned(out, parts, group)
