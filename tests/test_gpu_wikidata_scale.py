"""GPU parity at Wikidata scale (configs 4 and 5 of BASELINE.json): the 30M-node / 150M-edge
synthetic KG (WikiLarge-shaped), through the C-ABI, against the CPU oracle.

* config 4: the depth sweep D in {4, 6, 8, 10, 12, 16, 20} (max Glevel 20,
  P:637), 4 queries per depth from a 200-query batch (the 64-bit item loop), plus the full
  hitting-level and block arrays of both runs of one query;
* config 5: the bench's launch configuration -- a 1000-query chunk of the 10k throughput set
  (half 2 + 4, half the Exp-1 mix cknum x mknum in {1,2,4} x {2,4,6}) through the
  device batch path -- with 12 queries compared that span the mix, including |C| = 4 and
  |M| = 6 (64-bit rows).
The oracle runs its queries one per host thread (plain C behind ctypes)."""
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle as O
import synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def _cmp(dev, orc):
    assert len(dev.rpgs) == len(orc.rpgs), (len(dev.rpgs), len(orc.rpgs))
    for a, b in zip(dev.rpgs, orc.rpgs):
        assert (a.central_node, a.sc, a.sm, a.ptc, a.score) == (b.central_node, b.sc, b.sm, b.ptc, b.score)
        assert a.nodes.tolist() == b.nodes.tolist()
        assert a.edge_ids.tolist() == b.edge_ids.tolist()
        assert a.vc.tolist() == b.vc.tolist()
        assert a.cdist.tolist() == b.cdist.tolist() and a.mdist.tolist() == b.mdist.tolist()
    st = dev.stats
    assert (st["L_central"], st["L_marginal"], st["relax_central"], st["relax_marginal"]) == \
           (orc.Lc, orc.Lm, orc.relax_c, orc.relax_m)


@pytest.fixture(scope="module")
def wiki():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2001_06770_b200 as P
    kg = synth.make_kg(4)
    g = P.Graph(kg.n_nodes, kg.src, kg.dst, kg.label_class, kg.term_ptr, kg.postings)
    g.set_label_weights(0.5, kg.avg_hops)
    a = O.coarsen_all(O.fine_weights(kg.n_nodes, kg.src, kg.dst, kg.label_class), 0.5, kg.avg_hops)
    assert (g.activation_levels() == a).all()  # a2 at full size (R31 ln, Eq. 1-3)
    og = O.Graph(kg.n_nodes, kg.src, kg.dst, a)
    yield P, kg, g, og
    g.close()


def _oracle_many(kg, og, qs, idx, depth, threads=16):
    def one(i):
        return O.search(og, [kg.posting(t) for t in qs.central[i]], [kg.posting(t) for t in qs.marginal[i]], qs.k,
                        depth, want_matrices=False, want_candidates=False)
    with ThreadPoolExecutor(threads) as ex:
        return list(ex.map(one, idx))


def test_c4_depth_sweep(wiki):
    P, kg, g, og = wiki
    qs = synth.config_queries(kg, 4, 200)  # the bench batch: 200 x 30M > 2^32 items -> 64-bit loop
    picks = (0, 57, 131, 199)
    for depth in (4, 6, 8, 10, 12, 16, 20):
        res = g.search_batch(qs.central, qs.marginal, qs.k, depth)
        for i, ro in zip(picks, _oracle_many(kg, og, qs, picks, depth)):
            _cmp(res[i], ro)


def test_c4_full_matrices_one_query(wiki):
    # every cell of H and the block array of both runs (central CF, marginal stop rule)
    P, kg, g, og = wiki
    qs = synth.config_queries(kg, 4, 8)
    for terms, mode in ((qs.central[3], 1), (qs.marginal[3], 2)):
        H, blk, rel, L = g.hitting_levels(np.array(terms, np.uint32), 20, mode)
        Ho, bo, Lo, relo = O.phase(og, [kg.posting(t) for t in terms], 20, mode)
        assert (H == Ho).all() and (blk == bo).all() and rel == relo and L == Lo


def test_c5_bench_chunk_sampled(wiki):
    import torch
    P, kg, g, og = wiki
    qs = synth.config_queries(kg, 5)
    ids = list(range(1000))  # chunk 0 of the bench
    cs, ms = [qs.central[i] for i in ids], [qs.marginal[i] for i in ids]
    cp, ct = P.Graph._csr(cs)
    mp, mt = P.Graph._csr(ms)
    d = [torch.from_numpy(x.view(np.int64) if x.dtype == np.uint64 else x.view(np.int32)).cuda()
         for x in (cp, ct, mp, mt)]
    g.set_batch_slots(1000)
    g.search_batch_device(1000, *(x.data_ptr() for x in d), qs.k, qs.depth)
    res = g.fetch(1000, [len(c) for c in cs], [len(m) for m in ms])
    g.set_batch_slots(0)
    # 12 queries spanning the mix: the 2 + 4 half and every (cknum, mknum) of Exp-1 present
    shapes, picks = {}, []
    for i in ids:
        key = (len(cs[i]), len(ms[i]))
        if shapes.get(key, 0) < (4 if key == (2, 4) else 1):
            shapes[key] = shapes.get(key, 0) + 1
            picks.append(i)
    assert (4, 6) in shapes and (1, 2) in shapes and len(picks) >= 12, shapes
    for i, ro in zip(picks, _oracle_many(kg, og, qs, picks, qs.depth)):
        _cmp(res[i], ro)
