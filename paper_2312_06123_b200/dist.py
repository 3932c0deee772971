"""Multi-GPU plumbing: one process per GPU, queries sharded, results all-gathered.

The graph (CSR) is replicated on every rank; queries are independent,
so a rank answers its contiguous shard with ``query_index_base`` = the global index
of its first query -- the RNG streams, hence every output bit, do not depend on the
number of GPUs.  The only collective is one all-gather of the fp64 results
(torch.distributed; NCCL over NVLink on the GPU box, gloo in the CPU tests).
"""
from __future__ import annotations


def shard(k_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous balanced split of [0, k_total): rank r gets [lo, hi)."""
    if world < 1 or not (0 <= rank < world) or k_total < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(k_total, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


def gather_results(out_local, k_total: int, group=None):
    """All-gather every rank's fp64 results into a [k_total] tensor in global order.

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
