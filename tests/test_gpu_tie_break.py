"""GPU parity of the weight-sum tie-break (tie_break 1; "break the ties by a re-ranking
operation, e.g. using the sum of edge weights"; reading R29 in DESIGN.md §3): libriki.so
through the C-ABI against the CPU oracle, result order and identity bit for bit."""
import numpy as np
import pytest

import oracle as O
import synth
from fixtures import load_golden, random_instance

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2001_06770_b200 as pkg
    return pkg


def _graph(P, V, src, dst, post, w, alpha=0.5, avg=3.0):
    tp = np.zeros(len(post) + 1, np.uint64)
    tp[1:] = np.cumsum([len(x) for x in post])
    po = np.concatenate([np.asarray(x, np.uint32) for x in post])
    g = P.Graph(V, src, dst, None, tp, po)
    g.set_edge_weights(w, alpha, avg)
    return g


def _same(r, ro):
    assert [(x.central_node, x.sc, x.sm, x.score, x.ptc) for x in r.rpgs] == \
           [(x.central_node, x.sc, x.sm, x.score, x.ptc) for x in ro.rpgs]
    for a, b in zip(r.rpgs, ro.rpgs):
        assert a.nodes.tolist() == b.nodes.tolist() and a.edge_ids.tolist() == b.edge_ids.tolist()


def test_tie_break_golden_fixture(P):
    d = load_golden("tie_break_weight_sum.json")
    e = d["directed_edges"]
    src = np.array([x[0] for x in e], np.uint32)
    dst = np.array([x[1] for x in e], np.uint32)
    wf = np.array([x[2] for x in e], np.float64)
    # Abar = 0.2 keeps every coarsened activation at 0 (Eq. 1-3: a <= round(2 * 0.2) = 0)
    g = _graph(P, d["nodes"], src, dst, d["central"] + d["marginal"], wf, 0.5, 0.2)
    assert (g.activation_levels() == d["activation"]).all()
    for case in d["cases"]:
        M = [2] if case["marginal"] else []
        kw = dict(tie_break=case["tie_break"], beam_w=case.get("beam_w", 0), beam_mode=case.get("beam_mode", 0))
        r = g.search([0, 1], M, case["k"], d["depth"], **kw)
        assert [x.central_node for x in r.rpgs] == case["expect"], case
        for x, ed in zip(r.rpgs, case.get("edges", [])):
            assert x.edge_ids.tolist() == ed


@pytest.mark.parametrize("seed", range(40))
def test_tie_break_random(P, seed):
    rng = np.random.default_rng(12000 + seed)
    V, src, dst, _, _ = random_instance(rng, 10, 120, deg=2.6)
    wf = rng.integers(0, 9, len(src)) / 8.0  # coarse grid: ties on W happen too
    nterm = 8
    post = [np.unique(rng.integers(0, V, int(rng.integers(1, 5)))).astype(np.uint32) for _ in range(nterm)]
    A = float(rng.choice([0.6, 1.5, 3.0]))
    g = _graph(P, V, src, dst, post, wf, 0.5, A)
    og = O.Graph(V, src, dst, O.coarsen_all(wf, 0.5, A))  # oracle-computed activations (Eq. 1-3)
    for _ in range(4):
        nc = int(rng.integers(1, 4))
        nm = int(rng.integers(0, 4))
        tt = rng.choice(nterm, nc + nm, replace=False)
        C, M = tt[:nc], tt[nc:]
        k = int(rng.choice([1, 2, 3, 5, 8]))
        D = int(rng.choice([4, 20]))
        kw = dict(ptc_mode=int(rng.integers(0, 4)), early_term=int(rng.choice([0, 2])),
                  beam_mode=int(rng.integers(0, 2)), beam_w=int(rng.choice([0, k, k + 1, 2 * k])))
        r = g.search(C, M, k, D, tie_break=1, **kw)
        ro = O.search(og, [post[t] for t in C], [post[t] for t in M], k, D, tie_break=1, wfine=wf, **kw)
        _same(r, ro)


def test_tie_break_batch_and_node_weights(P):
    kg = synth.make_kg(1)
    qs = synth.config_queries(kg, 1)
    g = P.Graph(kg.n_nodes, kg.src, kg.dst, kg.label_class, kg.term_ptr, kg.postings)
    g.set_label_weights(0.5, kg.avg_hops)
    wf = O.fine_weights(kg.n_nodes, kg.src, kg.dst, kg.label_class)
    og = O.Graph(kg.n_nodes, kg.src, kg.dst, O.coarsen_all(wf, 0.5, kg.avg_hops))
    res = g.search_batch(qs.central, qs.marginal, qs.k, qs.depth, tie_break=1)
    for i, r in enumerate(res):
        ro = O.search(og, [kg.posting(t) for t in qs.central[i]], [kg.posting(t) for t in qs.marginal[i]], qs.k,
                      qs.depth, tie_break=1, wfine=wf)
        _same(r, ro)
    # node weights: the fine weight of edge f -> n is w[n]
    rng = np.random.default_rng(5)
    wn = rng.integers(0, 5, kg.n_nodes) / 4.0
    g.set_node_weights(wn, 0.5, kg.avg_hops)
    og = O.Graph(kg.n_nodes, kg.src, kg.dst, O.coarsen_all(wn[kg.dst], 0.5, kg.avg_hops))
    we = wn[kg.dst]
    for i in range(0, len(qs.central), 7):
        r = g.search(qs.central[i], qs.marginal[i], qs.k, qs.depth, tie_break=1)
        ro = O.search(og, [kg.posting(t) for t in qs.central[i]], [kg.posting(t) for t in qs.marginal[i]], qs.k,
                      qs.depth, tie_break=1, wfine=we)
        _same(r, ro)
    # exact activation levels carry no fine weights: the tie-break is refused
    g.set_activation_levels(g.activation_levels())
    with pytest.raises(P.RikiError) as ei:
        g.search(qs.central[0], qs.marginal[0], qs.k, qs.depth, tie_break=1)
    assert ei.value.code == -6  # RIKI_ENOWEIGHTS


@pytest.mark.slow
def test_tie_break_c2_sampled(P):
    kg = synth.make_kg(2)
    qs = synth.config_queries(kg, 2, 16)
    g = P.Graph(kg.n_nodes, kg.src, kg.dst, kg.label_class, kg.term_ptr, kg.postings)
    g.set_label_weights(0.5, kg.avg_hops)
    res = g.search_batch(qs.central, qs.marginal, qs.k, qs.depth, tie_break=1)
    wf = O.fine_weights(kg.n_nodes, kg.src, kg.dst, kg.label_class)
    og = O.Graph(kg.n_nodes, kg.src, kg.dst, O.coarsen_all(wf, 0.5, kg.avg_hops))
    for i in (0, 5, 11):
        ro = O.search(og, [kg.posting(t) for t in qs.central[i]], [kg.posting(t) for t in qs.marginal[i]], qs.k,
                      qs.depth, tie_break=1, wfine=wf, want_matrices=False)
        _same(res[i], ro)
