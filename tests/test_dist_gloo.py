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
