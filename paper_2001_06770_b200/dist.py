"""Multi-GPU plumbing for the RIKI hot path.

RPQ queries are independent units, so the path shards by query: the graph is replicated on
every GPU (one process per GPU, torch.distributed), each rank runs its contiguous shard of
the batch through libriki.so, and the only collective is the gather of the (small) result
sets, plus the max-over-ranks timing reduction of the benchmark.  No collective touches the
data path.  Everything here is host logic, covered by world_size-2 gloo tests on CPU."""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def shard(n: int, rank: int, world: int) -> tuple[int, int]:
    """Balanced contiguous shard [lo, hi) of n queries for `rank` of `world`."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def search_sharded(search_fn, centrals, marginals, k, depth, group=None, **kw):
    """Run search_fn(centrals_shard, marginals_shard, k, depth, **kw) on this rank's shard and
    all-gather the per-query results (pickled, via the process group); every rank returns the
    full list in the original query order."""
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    lo, hi = shard(len(centrals), rank, world)
    local = search_fn(centrals[lo:hi], marginals[lo:hi], k, depth, **kw) if hi > lo else []
    parts = [None] * world
    dist.all_gather_object(parts, local, group=group)
    return [r for p in parts for r in p]


_FIELDS = ("cnt", "hdr", "score", "nodes", "edges", "vc", "cd", "md", "stats")


def pack_batch(br) -> np.ndarray:
    """A BatchResult's columnar arrays as one byte buffer: a u64 header (n, then per field the
    byte length) followed by the raw arrays (query term counts travel in the stats)."""
    arrs = [np.ascontiguousarray(getattr(br, f)) for f in _FIELDS]
    hdr = np.array([br.n, len(br.ncs)] + list(br.ncs) + list(br.nms) + [a.nbytes for a in arrs], np.uint64)
    return np.concatenate([hdr.view(np.uint8)] + [a.reshape(-1).view(np.uint8) for a in arrs])


def unpack_batch(buf: np.ndarray, like):
    """Inverse of pack_batch; `like` supplies dtypes / trailing shapes (any BatchResult)."""
    from .riki import BatchResult
    buf = np.ascontiguousarray(buf, np.uint8)
    n, m = (int(x) for x in buf[:16].view(np.uint64))
    ncs = [int(x) for x in buf[16:16 + 8 * m].view(np.uint64)]
    nms = [int(x) for x in buf[16 + 8 * m:16 + 16 * m].view(np.uint64)]
    o = 16 + 16 * m
    lens = [int(x) for x in buf[o:o + 8 * len(_FIELDS)].view(np.uint64)]
    o += 8 * len(_FIELDS)
    out = {}
    for f, ln in zip(_FIELDS, lens):
        ref = getattr(like, f)
        a = buf[o:o + ln].view(ref.dtype)
        out[f] = a.reshape((-1,) + ref.shape[1:]) if ref.ndim > 1 else a
        o += ln
    return BatchResult(n, ncs, nms, out["cnt"], out["hdr"], out["score"], out["nodes"], out["edges"], out["vc"],
                       out["cd"], out["md"], out["stats"][:n])


def gather_results(br, group=None, device=None):
    """Gather every rank's BatchResult to rank 0 over the process group (the one
    exchange of the replicated mode).  The packed buffers are padded to the largest and
    all-gathered as one tensor on `device` (NCCL over NVLink on GPUs; gloo on CPU).  Returns
    the list of per-rank BatchResults on rank 0 (rank order = query-shard order), None elsewhere."""
    import torch
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    buf = pack_batch(br)
    n = torch.tensor([buf.size], dtype=torch.int64, device=device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    mx = int(max(int(x.item()) for x in sizes))
    t = torch.zeros(mx, dtype=torch.uint8, device=device)
    t[:buf.size] = torch.from_numpy(buf).to(t.device)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t, group=group)
    if rank != 0:
        return None
    return [unpack_batch(p[:int(sz.item())].cpu().numpy(), br) for p, sz in zip(parts, sizes)]


def init_vertex_partitioned(graph, group=None, unique_id_fn=None):
    """Vertex-partitioned mode over the ranks of `group`: rank 0 draws the NCCL
    unique id (riki_dist_unique_id), the process group broadcasts it, and every rank binds its
    graph handle to one NCCL communicator (riki_dist_init, mode 1).  Every rank then issues the
    same searches; each gets the identical result.  Returns (rank, world)."""
    from .riki import dist_unique_id
    rank = dist.get_rank(group)
    world = dist.get_world_size(group)
    uid = [(unique_id_fn or dist_unique_id)() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    graph.dist_init(world, rank, uid[0], mode=1)
    return rank, world


def max_over_ranks(x: float, group=None, device=None) -> float:
    """Max of a host float over the ranks (NCCL needs a CUDA tensor, gloo a CPU one)."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sum_over_ranks(x: float, group=None, device=None) -> float:
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return float(t.item())
