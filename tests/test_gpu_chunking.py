"""Batches whose recovery arena (memoised Alg. 2 predecessor lists + recovered subgraphs,
32-bit offsets) would overflow run in chunks of fewer queries -- host batch and device batch
paths give the unchunked results.  A small riki_set_arena_limit forces the chunking."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2001_06770_b200 as pkg
    return pkg


def _key(res):
    return [[(x.central_node, x.sc, x.sm, x.score, x.nodes.tolist(), x.edge_ids.tolist()) for x in r.rpgs] for r in res]


def _graph(P, kg):
    g = P.Graph(kg.n_nodes, kg.src, kg.dst, kg.label_class, kg.term_ptr, kg.postings)
    g.set_label_weights(0.5, kg.avg_hops)
    return g


def test_arena_limit_chunks_host_and_device_batches(P):
    import torch
    kg = synth.make_kg(1)
    qs = synth.config_queries(kg, 1)
    base = _key(_graph(P, kg).search_batch(qs.central, qs.marginal, qs.k, qs.depth))
    cp, ct = P.Graph._csr(qs.central)
    mp, mt = P.Graph._csr(qs.marginal)
    d = [torch.from_numpy(x.view(np.int64) if x.dtype == np.uint64 else x.view(np.int32)).cuda() for x in (cp, ct, mp, mt)]
    chunked = 0
    for limit in (1 << 14, 1 << 12):
        g = _graph(P, kg)
        g.set_arena_limit(limit)
        g.reset_stats()
        try:
            got = g.search_batch(qs.central, qs.marginal, qs.k, qs.depth)
        except P.RikiError as e:  # a single query needs more than the limit
            assert e.code == -2
            continue
        assert _key(got) == base
        chunked += g.stats()["retries"] > 0
        g2 = _graph(P, kg)
        g2.set_arena_limit(limit)
        n = len(qs.central)
        g2.search_batch_device(n, *(x.data_ptr() for x in d), qs.k, qs.depth)
        assert _key(g2.fetch(n, [len(c) for c in qs.central], [len(m) for m in qs.marginal])) == base
    assert chunked >= 1


def test_wide_item_indexing_matches(P, monkeypatch):
    # k_expand's 64-bit item loop (batches with > 2^32 frontier items per level) forced on a
    # small batch gives the 32-bit loop's results
    kg = synth.make_kg(1)
    qs = synth.config_queries(kg, 1)
    g = _graph(P, kg)
    base = _key(g.search_batch(qs.central, qs.marginal, qs.k, qs.depth))
    monkeypatch.setenv("RIKI_FORCE_WIDE", "1")
    assert _key(g.search_batch(qs.central, qs.marginal, qs.k, qs.depth)) == base


def test_load_graph_device_matches_host_load(P):
    import torch
    kg = synth.make_kg(1)
    qs = synth.config_queries(kg, 1)
    host = _graph(P, kg)
    base = _key(host.search_batch(qs.central, qs.marginal, qs.k, qs.depth))
    t = [torch.from_numpy(np.ascontiguousarray(x).view(np.int32)).cuda() for x in (kg.src, kg.dst, kg.label_class)]
    tp = torch.from_numpy(np.ascontiguousarray(kg.term_ptr, np.uint64).view(np.int64)).cuda()
    po = torch.from_numpy(np.ascontiguousarray(kg.postings, np.uint32).view(np.int32)).cuda()
    g = P.Graph.from_device(kg.n_nodes, len(kg.src), t[0].data_ptr(), t[1].data_ptr(), t[2].data_ptr(),
                            len(kg.term_ptr) - 1, tp.data_ptr(), po.data_ptr())
    del t, tp, po  # copied: the caller may free its arrays
    torch.cuda.synchronize()
    g.set_label_weights(0.5, kg.avg_hops)
    assert (g.activation_levels() == host.activation_levels()).all()
    assert _key(g.search_batch(qs.central, qs.marginal, qs.k, qs.depth)) == base
    # device-side validation
    bad = torch.from_numpy(np.ascontiguousarray(kg.dst).view(np.int32)).cuda()
    bad[3] = kg.n_nodes
    good = torch.from_numpy(np.ascontiguousarray(kg.src).view(np.int32)).cuda()
    tp = torch.from_numpy(np.ascontiguousarray(kg.term_ptr, np.uint64).view(np.int64)).cuda()
    po = torch.from_numpy(np.ascontiguousarray(kg.postings, np.uint32).view(np.int32)).cuda()
    with pytest.raises(P.RikiError) as ei:
        P.Graph.from_device(kg.n_nodes, len(kg.src), good.data_ptr(), bad.data_ptr(), 0, len(kg.term_ptr) - 1,
                            tp.data_ptr(), po.data_ptr())
    assert ei.value.code == -1


def test_level_graphs_match_plain_launches(P, monkeypatch):
    # the level loop replayed as CUDA graphs (default) and as plain launches give the same
    # results, over repeated calls (graph cache hits) and changing batch shapes
    kg = synth.make_kg(1)
    qs = synth.config_queries(kg, 1)
    g = _graph(P, kg)
    monkeypatch.setenv("RIKI_NO_GRAPHS", "1")
    plain = _key(g.search_batch(qs.central, qs.marginal, qs.k, qs.depth))
    single = [_key([g.search(qs.central[i], qs.marginal[i], qs.k, qs.depth)]) for i in range(8)]
    H0 = g.hitting_levels(np.arange(3, dtype=np.uint32), 20, 1)
    monkeypatch.delenv("RIKI_NO_GRAPHS")
    for chunked in (False, True):  # whole-run graph (device while loop) / 4-level chunk graphs
        if chunked:
            monkeypatch.setenv("RIKI_CHUNK_GRAPHS", "1")
        for _ in range(2):
            assert _key(g.search_batch(qs.central, qs.marginal, qs.k, qs.depth)) == plain
            assert [_key([g.search(qs.central[i], qs.marginal[i], qs.k, qs.depth)]) for i in range(8)] == single
        H1 = g.hitting_levels(np.arange(3, dtype=np.uint32), 20, 1)
        assert all((a == b).all() if hasattr(a, "all") else a == b for a, b in zip(H0, H1))
        for D in (0, 1, 3):  # depth bounds around the loop's exit rule
            monkeypatch.setenv("RIKI_NO_GRAPHS", "1")
            ref = _key(g.search_batch(qs.central, qs.marginal, qs.k, D))
            monkeypatch.delenv("RIKI_NO_GRAPHS")
            assert _key(g.search_batch(qs.central, qs.marginal, qs.k, D)) == ref


@pytest.mark.timeout(600)
def test_bench_two_ranks_replicated_gloo(P):
    # bench.py's multi-rank path (torchrun, weak scaling, max over ranks) with two ranks sharing
    # the pool's one GPU (gloo for the plumbing; the contract run uses NCCL, one GPU per rank)
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, RIKI_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2", "--master-addr",
           "127.0.0.1", "--master-port", "29517", "bench.py", "--gpus", "2", "--config", "1", "--steps", "2",
           "--warmup", "3", "--no-cpu", "--latency-queries", "2"]
    out = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=500)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0 and d["gpu_launches"] > 0


@pytest.mark.parametrize("seed", range(16))
def test_modes_combined_against_oracle(P, seed, monkeypatch):
    # every search mode combined with every execution variant (plain launches / whole-run graph /
    # 64-bit item loop / simulated vertex partitions) gives the oracle's results
    import oracle as O
    from fixtures import random_instance
    rng = np.random.default_rng(13000 + seed)
    V, src, dst, _, _ = random_instance(rng, 20, 150, deg=2.8)
    wf = rng.integers(0, 9, len(src)) / 8.0
    nterm = 8
    post = [np.unique(rng.integers(0, V, int(rng.integers(1, 5)))).astype(np.uint32) for _ in range(nterm)]
    tp = np.zeros(nterm + 1, np.uint64)
    tp[1:] = np.cumsum([len(x) for x in post])
    g = P.Graph(V, src, dst, None, tp, np.concatenate(post))
    A = float(rng.choice([1.0, 2.0, 3.5]))
    g.set_edge_weights(wf, 0.5, A)
    og = O.Graph(V, src, dst, O.coarsen_all(wf, 0.5, A))  # oracle-computed activations (Eq. 1-3)
    variant = seed % 4
    if variant == 0:
        monkeypatch.setenv("RIKI_NO_GRAPHS", "1")
    elif variant == 2:
        monkeypatch.setenv("RIKI_FORCE_WIDE", "1")
    elif variant == 3:
        g.dist_init(int(rng.choice([2, 3, 5])), 0, None, mode=1)
    cs, ms, kws, refs = [], [], [], []
    k = int(rng.choice([1, 3, 5]))
    D = int(rng.choice([3, 8, 20]))
    kw = dict(ptc_mode=int(rng.integers(0, 4)), early_term=int(rng.integers(0, 3)), beam_mode=int(rng.integers(0, 2)),
              tie_break=int(rng.integers(0, 2)))
    for _ in range(6):
        nc = int(rng.integers(1, 4))
        nm = int(rng.integers(0, 4))
        tt = rng.choice(nterm, nc + nm, replace=False)
        cs.append([int(x) for x in tt[:nc]])
        ms.append([int(x) for x in tt[nc:]])
        refs.append(O.search(og, [post[t] for t in cs[-1]], [post[t] for t in ms[-1]], k, D, wfine=wf, **kw))
    res = g.search_batch(cs, ms, k, D, **kw)
    for r, ro in zip(res, refs):
        assert [(x.central_node, x.sc, x.sm, x.score, x.ptc, x.edge_ids.tolist()) for x in r.rpgs] == \
               [(x.central_node, x.sc, x.sm, x.score, x.ptc, x.edge_ids.tolist()) for x in ro.rpgs]
