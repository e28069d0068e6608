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
