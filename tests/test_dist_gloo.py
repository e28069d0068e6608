"""world_size-2 gloo tests of the multi-GPU host logic (query sharding, result gather,
max-over-ranks timing) on CPU.  The per-rank search is the CPU oracle standing in for the
GPU (the sharding logic is identical), so the gathered answer must equal one process."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2001_06770_b200.dist import max_over_ranks, search_sharded, shard, sum_over_ranks


def test_shard_covers_and_balances():
    for n in range(0, 40):
        for world in (1, 2, 3, 8):
            parts = [shard(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [h - l for l, h in parts]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_search_fn(kg, og):
    import oracle as O

    def fn(cs, ms, k, depth):
        out = []
        for c, m in zip(cs, ms):
            r = O.search(og, [kg.posting(t) for t in c], [kg.posting(t) for t in m], k, depth,
                         want_matrices=False, want_candidates=False)
            out.append([(x.central_node, x.sc, x.sm, x.score, x.nodes.tolist(), x.edge_ids.tolist()) for x in r.rpgs])
        return out
    return fn


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle as O
    import synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        kg = synth.make_kg(1)
        qs = synth.config_queries(kg, 1, 21)  # odd count: uneven shards
        og = O.Graph(kg.n_nodes, kg.src, kg.dst,
                     O.coarsen_all(O.fine_weights(kg.n_nodes, kg.src, kg.dst, kg.label_class), 0.5, kg.avg_hops))
        res = search_sharded(_oracle_search_fn(kg, og), qs.central, qs.marginal, qs.k, qs.depth)
        t = max_over_ranks(float(rank + 1))
        s = sum_over_ranks(float(rank + 1))
        q.put((rank, res, t, s))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_search_sharded_gloo_world2_matches_single_process():
    import oracle as O
    import synth
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    kg = synth.make_kg(1)
    qs = synth.config_queries(kg, 1, 21)
    og = O.Graph(kg.n_nodes, kg.src, kg.dst,
                 O.coarsen_all(O.fine_weights(kg.n_nodes, kg.src, kg.dst, kg.label_class), 0.5, kg.avg_hops))
    ref = _oracle_search_fn(kg, og)(qs.central, qs.marginal, qs.k, qs.depth)
    for rank, res, t, s in outs:
        assert res == ref               # every rank holds the full, ordered answer
        assert t == float(world)        # max over ranks
        assert s == float(world * (world + 1) // 2)


def _fake_batch(seed):
    """A BatchResult with random but consistent columnar content (no device needed)."""
    from paper_2001_06770_b200.riki import _STATS_DT, BatchResult
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 6))
    cnt = rng.integers(0, 3, n).astype(np.uint32)
    nr = int(cnt.sum())
    hdr = np.zeros((max(nr, 1), 8), np.uint32)
    hdr[:nr, :4] = rng.integers(0, 100, (nr, 4))
    hdr[:nr, 4:7] = rng.integers(0, 5, (nr, 3))
    sizes = hdr[:nr, 4:7].sum(axis=0) if nr else np.zeros(3, np.int64)
    score = rng.random(max(nr, 1))
    nodes = rng.integers(0, 1000, max(int(sizes[0]), 1)).astype(np.uint32)
    edges = rng.integers(0, 5000, max(int(sizes[1]), 1)).astype(np.uint64)
    vc = rng.integers(0, 1000, max(int(sizes[2]), 1)).astype(np.uint32)
    cd = rng.integers(0, 9, (max(nr, 1), 8)).astype(np.uint8)
    md = rng.integers(0, 9, (max(nr, 1), 8)).astype(np.uint8)
    stats = np.zeros(n, dtype=_STATS_DT)
    for f in _STATS_DT.names:
        stats[f] = rng.integers(0, 50, n)
    ncs = [int(x) for x in rng.integers(1, 4, n)]
    nms = [int(x) for x in rng.integers(0, 4, n)]
    return BatchResult(n, ncs, nms, cnt, hdr, score, nodes, edges, vc, cd, md, stats)


def _flat(br):
    return [([(x.central_node, x.sc, x.sm, x.score, x.ptc, x.nodes.tolist(), x.edge_ids.tolist(), x.vc.tolist(),
               x.cdist.tolist(), x.mdist.tolist()) for x in r.rpgs], sorted(r.stats.items())) for r in br]


def _gather_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2001_06770_b200.dist import gather_results
        got = gather_results(_fake_batch(100 + rank))
        q.put((rank, None if got is None else [_flat(b) for b in got]))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_gather_results_gloo_world2():
    # the replicated mode's one exchange: every rank's columnar results reach rank 0 intact
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert outs[1] is None
    assert outs[0] == [_flat(_fake_batch(100 + r)) for r in range(world)]


def test_pack_unpack_roundtrip():
    from paper_2001_06770_b200.dist import pack_batch, unpack_batch
    for seed in range(10):
        b = _fake_batch(seed)
        assert _flat(unpack_batch(pack_batch(b), b)) == _flat(b)
