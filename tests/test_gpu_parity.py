"""GPU parity: libriki.so (through the C-ABI) against the CPU oracle, element by element.

Bar (BASELINE.json north star): bit-exact activation levels, hitting levels, block levels,
candidate CG sets, result identity (central node, node set, edge-id set, V_C, distances),
relaxation counts; scores compared exactly (same fp64 expression order; tolerance 1e-6
relative would also be acceptable per the north star, the test asserts equality)."""
import numpy as np
import pytest

import oracle as O
import synth
from fixtures import load_golden, random_instance, undirected_to_directed

pytestmark = pytest.mark.gpu

INF = 0xFF


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2001_06770_b200 as pkg
    return pkg


def _dev_graph(P, V, src, dst, act, postings, cls=None):
    """postings: list of node lists; returns device graph with activations set exactly."""
    tp = np.zeros(len(postings) + 1, np.uint64)
    tp[1:] = np.cumsum([len(x) for x in postings])
    po = np.concatenate([np.asarray(x, np.uint32) for x in postings]) if postings else np.zeros(0, np.uint32)
    g = P.Graph(V, src, dst, cls, tp, po)
    g.set_activation_levels(act)
    return g


def _cmp_results(dev, orc, src=None, dst=None):
    assert len(dev.rpgs) == len(orc.rpgs), (len(dev.rpgs), len(orc.rpgs))
    for a, b in zip(dev.rpgs, orc.rpgs):
        assert (a.central_node, a.sc, a.sm, a.ptc) == (b.central_node, b.sc, b.sm, b.ptc)
        assert a.score == b.score
        assert a.nodes.tolist() == b.nodes.tolist()
        assert a.edge_ids.tolist() == b.edge_ids.tolist()
        assert a.vc.tolist() == b.vc.tolist()
        assert a.cdist.tolist() == b.cdist.tolist()
        assert a.mdist.tolist() == b.mdist.tolist()


# ---------------------------------------------------------------- activation levels (a2)
def test_label_weights_match_oracle_c1(P):
    kg = synth.make_kg(1)
    g = P.Graph(kg.n_nodes, kg.src, kg.dst, kg.label_class, kg.term_ptr, kg.postings)
    g.set_label_weights(0.5, kg.avg_hops)
    w = O.fine_weights(kg.n_nodes, kg.src, kg.dst, kg.label_class)
    assert (g.activation_levels() == O.coarsen_all(w, 0.5, kg.avg_hops)).all()


def test_edge_and_node_weights_match_oracle(P):
    rng = np.random.default_rng(77)
    V, src, dst, act, terms = random_instance(rng, 50, 300)
    g = _dev_graph(P, V, src, dst, act, terms)
    for alpha in (0.2, 0.5, 0.8):
        for A in (2.0, 3.68, 3.87, 5.5):
            w = rng.random(len(src))
            w[:5] = [0.0, 1.0, alpha, 0.5, 0.25]
            g.set_edge_weights(w, alpha, A)
            assert (g.activation_levels() == O.coarsen_all(w, alpha, A)).all()
            wn = rng.random(V)
            g.set_node_weights(wn, alpha, A)
            assert (g.activation_levels() == O.coarsen_all(wn[dst], alpha, A)).all()


# ---------------------------------------------------------------- hitting levels (a3-a5)
@pytest.mark.parametrize("seed", range(30))
def test_hitting_levels_random(P, seed):
    rng = np.random.default_rng(3000 + seed)
    V, src, dst, act, terms = random_instance(rng, 5, 300, deg=3.0, T_hi=8, post_hi=6)
    g = _dev_graph(P, V, src, dst, act, terms)
    og = O.Graph(V, src, dst, act)
    D = int(rng.choice([0, 1, 3, 5, 20]))
    T = len(terms)
    for mode in (0, 1, 2):
        H, blk, rel, L = g.hitting_levels(np.arange(T, dtype=np.uint32), D, mode)
        Ho, bo, Lo, relo = O.phase(og, terms, D, mode)
        assert (H == Ho).all(), (mode, np.argwhere(H != Ho)[:5])
        assert (blk == bo).all()
        assert L == Lo and rel == relo


@pytest.mark.parametrize("seed", range(10))
def test_expansion_counters_against_oracle(P, seed):
    # the device counters behind the bench's SURVEY §8(d) byte model and random-access roofline:
    # new cells = the oracle's finite non-seed cells of H exactly; every walked edge relaxes 1..T
    # columns (P_e <= R <= T * P_e, R the oracle's relaxation count); every relaxation atomic
    # turns 1..T cells (or loses a race) and follows one walked edge (cells / T <= atomics <= P_e)
    rng = np.random.default_rng(3300 + seed)
    V, src, dst, act, terms = random_instance(rng, 20, 300, deg=4.0, T_hi=8, post_hi=6)
    g = _dev_graph(P, V, src, dst, act, terms)
    g.set_profiling(True)  # the atomics are counted by the profiling-mode kernels
    og = O.Graph(V, src, dst, act)
    T = len(terms)
    for mode in (0, 1, 2):
        g.reset_stats()
        H, blk, rel, L = g.hitting_levels(np.arange(T, dtype=np.uint32), 20, mode)
        Ho, bo, Lo, relo = O.phase(og, terms, 20, mode)
        assert (H == Ho).all() and rel == relo
        st = g.stats()
        cells = int(((Ho > 0) & (Ho < INF)).sum())
        assert st["exp_new_cells"] == cells, (st["exp_new_cells"], cells)
        pe, atoms = st["exp_edges"], st["exp_atomics"]
        assert pe <= relo <= T * pe, (pe, relo, T)
        assert -(-cells // T) <= atoms <= pe, (cells, atoms, pe)


@pytest.mark.parametrize("seed", range(12))
def test_hitting_levels_long_rows_high_activations(P, seed):
    """Rows longer than 8 edges with activations past the gate offset table (a >= 16): the table
    lookup and the binary search above it must give the oracle's hitting levels (Alg. 1 gate)."""
    rng = np.random.default_rng(3500 + seed)
    V, src, dst, act, terms = random_instance(rng, 20, 160, deg=14.0, amax=40, T_hi=5, post_hi=4)
    g = _dev_graph(P, V, src, dst, act, terms)
    og = O.Graph(V, src, dst, act)
    T = len(terms)
    for D in (7, 17, 60):
        for mode in (0, 1, 2):
            H, blk, rel, L = g.hitting_levels(np.arange(T, dtype=np.uint32), D, mode)
            Ho, bo, Lo, relo = O.phase(og, terms, D, mode)
            assert (H == Ho).all(), (D, mode, np.argwhere(H != Ho)[:5])
            assert (blk == bo).all() and L == Lo and rel == relo


@pytest.mark.parametrize("seed", range(8))
def test_search_long_rows_high_activations(P, seed):
    rng = np.random.default_rng(5500 + seed)
    V, src, dst, act, _ = random_instance(rng, 30, 120, deg=12.0, amax=30)
    nterm = 8
    post = [np.unique(rng.integers(0, V, int(rng.integers(1, 4)))).astype(np.uint32) for _ in range(nterm)]
    g = _dev_graph(P, V, src, dst, act, post)
    og = O.Graph(V, src, dst, act)
    for _ in range(3):
        nc = int(rng.integers(1, 3))
        nm = int(rng.integers(1, 3))
        tt = rng.choice(nterm, nc + nm, replace=False)
        C, M = tt[:nc], tt[nc:]
        r = g.search(C, M, 5, 60)
        ro = _oracle_run(og, lambda t: post[t], C, M, 5, 60)
        _cmp_results(r, ro)
        assert r.stats["relax_central"] == ro.relax_c and r.stats["relax_marginal"] == ro.relax_m


def _double_entry_graph(V=48):
    """Every node is both retained (pending a = 30 edge) and newly reached at level 2, so the
    level-2 frontier holds ~2V entries (one retained + one new per node)."""
    src, dst, act = [], [], []
    for i in range(2, V):
        src += [0, 1, i]; dst += [i, i, 2 + (i - 1) % (V - 2)]; act += [0, 1, 30]
    return V, np.array(src, np.uint32), np.array(dst, np.uint32), np.array(act, np.uint8)


def test_frontier_queue_overflow_retried(P):
    """A level queue may need 2V entries (Alg. 1 lines 9-11 retention + first-writer enqueue):
    the overflow is detected, the queues regrow to 2V, and the answer equals the oracle's."""
    V, src, dst, act = _double_entry_graph()
    terms = [np.array([0], np.uint32), np.array([1], np.uint32)]
    g = _dev_graph(P, V, src, dst, act, terms)
    og = O.Graph(V, src, dst, act)
    g.reset_stats()
    for mode in (0, 1, 2):
        H, blk, rel, L = g.hitting_levels(np.arange(2, dtype=np.uint32), 40, mode)
        Ho, bo, Lo, relo = O.phase(og, terms, 40, mode)
        assert (H == Ho).all() and (blk == bo).all() and L == Lo and rel == relo
    assert g.stats()["retries"] >= 1
    g2 = _dev_graph(P, V, src, dst, act, terms)
    r = g2.search([0], [1], 3, 40)
    ro = _oracle_run(og, lambda t: terms[t], [0], [1], 3, 40)
    _cmp_results(r, ro)
    assert r.stats["relax_central"] == ro.relax_c and r.stats["relax_marginal"] == ro.relax_m


def test_hitting_levels_c1_all_terms(P):
    kg = synth.make_kg(1)
    g = P.Graph(kg.n_nodes, kg.src, kg.dst, kg.label_class, kg.term_ptr, kg.postings)
    g.set_label_weights(0.5, kg.avg_hops)
    og = O.Graph(kg.n_nodes, kg.src, kg.dst, _oracle_act(kg))
    for t0 in range(0, kg.n_terms - 4, 4):
        terms = np.arange(t0, t0 + 4, dtype=np.uint32)
        for mode in (0, 1, 2):
            H, blk, rel, L = g.hitting_levels(terms, 20, mode)
            Ho, bo, Lo, relo = O.phase(og, [kg.posting(t) for t in terms], 20, mode)
            assert (H == Ho).all() and (blk == bo).all() and rel == relo and L == Lo


# ---------------------------------------------------------------- full search (a6-a13)
@pytest.mark.parametrize("name", ["five_node.json", "diamond.json", "r16_blocked_relay.json",
                                  "ptc_fail_m2.json", "ptc_fail_m3.json", "ptc_pass_vc_marginal.json"])
def test_golden_fixtures(P, name):
    d = load_golden(name)
    s, t, a = undirected_to_directed(d["undirected_edges"])
    terms = d["central"] + d["marginal"]
    g = _dev_graph(P, d["nodes"], s, t, a, terms)
    nc = len(d["central"])
    r = g.search(np.arange(nc), np.arange(nc, len(terms)), d["k"], d["depth"], gamma=d["gamma"])
    assert len(r.rpgs) == len(d["expect"])
    for got, exp in zip(r.rpgs, d["expect"]):
        assert got.central_node == exp["central_node"] and got.sc == exp["sc"] and got.sm == exp["sm"]
        assert got.score == exp["score"]
        assert got.nodes.tolist() == exp["nodes"]
        assert sorted((int(s[e]), int(t[e])) for e in got.edge_ids) == sorted(tuple(x) for x in exp["directed_edges"])
    if "expect_ptc_fail" in d:
        assert r.stats["n_ptc_fail"] == d["expect_ptc_fail"]


@pytest.mark.parametrize("name", ["ptc_gm_only_r20i.json", "ptc_single_marginal_node.json",
                                  "early_term_literal_gamma1.json"])
def test_golden_mode_fixtures(P, name):
    # the hand-derived option fixtures (ptc_mode 2, R19', early_term 1 at gamma = 1) through the C-ABI
    d = load_golden(name)
    s, t, a = undirected_to_directed(d["undirected_edges"])
    terms = d["central"] + d["marginal"]
    g = _dev_graph(P, d["nodes"], s, t, a, terms)
    nc = len(d["central"])
    for run in d["runs"]:
        r = g.search(np.arange(nc), np.arange(nc, len(terms)), d["k"], d["depth"], gamma=d["gamma"], **run["params"])
        assert len(r.rpgs) == len(run["expect"]), run["params"]
        for got, exp in zip(r.rpgs, run["expect"]):
            assert (got.central_node, got.sc, got.sm, got.score, int(got.ptc)) == \
                   (exp["central_node"], exp["sc"], exp["sm"], exp["score"], exp["ptc"])
            assert got.nodes.tolist() == exp["nodes"]
            assert sorted((int(s[e]), int(t[e])) for e in got.edge_ids) == \
                   sorted(tuple(x) for x in exp["directed_edges"])
        if "expect_ptc_fail" in run:
            assert r.stats["n_ptc_fail"] == run["expect_ptc_fail"]
        if "expect_L_marginal" in run:
            assert r.stats["L_marginal"] == run["expect_L_marginal"]


def _oracle_act(kg, alpha=0.5):
    """Activation levels computed by the ORACLE from the label-class fine weights:
    the oracle never takes an input produced by the CUDA path."""
    return O.coarsen_all(O.fine_weights(kg.n_nodes, kg.src, kg.dst, kg.label_class), alpha, kg.avg_hops)


def _oracle_run(og, kg_post, C, M, k, D, **kw):
    return O.search(og, [kg_post(t) for t in C], [kg_post(t) for t in M], k, D, **kw)


@pytest.mark.parametrize("seed", range(60))
def test_search_random_small(P, seed):
    rng = np.random.default_rng(5000 + seed)
    V, src, dst, act, _ = random_instance(rng, 6, 60, deg=2.5, amax=4)
    nterm = 10
    post = [np.unique(rng.integers(0, V, int(rng.integers(1, 4)))).astype(np.uint32) for _ in range(nterm)]
    g = _dev_graph(P, V, src, dst, act, post)
    g.set_debug(True)
    og = O.Graph(V, src, dst, act)
    for _ in range(4):
        nc = int(rng.integers(1, 4))
        nm = int(rng.integers(0, 4))
        tt = rng.choice(nterm, nc + nm, replace=False)
        C, M = tt[:nc], tt[nc:]
        k = int(rng.choice([1, 3, 5]))
        D = int(rng.choice([3, 6, 20]))
        kw = dict(ptc_mode=int(rng.integers(0, 4)), early_term=int(rng.integers(0, 3)),
                  beam_mode=int(rng.integers(0, 2)))
        r = g.search(C, M, k, D, **kw)
        ro = _oracle_run(og, lambda t: post[t], C, M, k, D, **kw)
        _cmp_results(r, ro)
        assert r.candidates == [(c.sc, c.v) for c in ro.candidates]
        assert r.stats["L_central"] == ro.Lc and r.stats["L_marginal"] == ro.Lm
        assert r.stats["relax_central"] == ro.relax_c and r.stats["relax_marginal"] == ro.relax_m
        # the GPU recovers an attached candidate's RPG (and checks its PTC) only if the candidate
        # can still enter the top-k (bounded recovery); the oracle checks every attached one
        assert r.stats["n_attached"] == ro.n_attached and r.stats["n_ptc_fail"] <= ro.n_ptc_fail


@pytest.mark.parametrize("seed", range(12))
def test_bounded_rpg_recovery_equals_eager(P, seed, monkeypatch):
    # bounded recovery (only candidates that can still enter the top-k get their RPG and PTC)
    # returns exactly what eager recovery of every attached candidate returns; eager recovery
    # also reproduces the oracle's PTC-failure count
    rng = np.random.default_rng(15000 + seed)
    V, src, dst, act, _ = random_instance(rng, 20, 120, deg=2.6, amax=3)
    nterm = 8
    post = [np.unique(rng.integers(0, V, int(rng.integers(1, 5)))).astype(np.uint32) for _ in range(nterm)]
    g = _dev_graph(P, V, src, dst, act, post)
    og = O.Graph(V, src, dst, act)
    Cs, Ms = [], []
    for _ in range(16):
        nc, nm = int(rng.integers(1, 3)), int(rng.integers(1, 4))
        tt = rng.choice(nterm, nc + nm, replace=False)
        Cs.append(tt[:nc].tolist())
        Ms.append(tt[nc:].tolist())
    k = int(rng.choice([1, 2, 4]))
    kw = dict(ptc_mode=int(rng.choice([0, 1, 2])))
    monkeypatch.setenv("RIKI_BOUNDED_RPG", "1")  # (the library picks it by itself for large candidate sets)
    bounded = g.search_batch(Cs, Ms, k, 20, **kw)
    monkeypatch.delenv("RIKI_BOUNDED_RPG")
    monkeypatch.setenv("RIKI_EAGER_RPG", "1")
    eager = g.search_batch(Cs, Ms, k, 20, **kw)
    for i, (a, b) in enumerate(zip(bounded, eager)):
        _cmp_results(a, b)
        ro = _oracle_run(og, lambda t: post[t], Cs[i], Ms[i], k, 20, **kw)
        _cmp_results(a, ro)
        assert b.stats["n_ptc_fail"] == ro.n_ptc_fail and b.stats["n_attached"] == ro.n_attached
        assert a.stats["n_ptc_fail"] <= b.stats["n_ptc_fail"]
        assert (a.stats["L_marginal"], a.stats["relax_marginal"]) == (b.stats["L_marginal"], b.stats["relax_marginal"])


def test_search_batch_c1_all_queries(P):
    kg = synth.make_kg(1)
    qs = synth.config_queries(kg, 1)
    g = P.Graph(kg.n_nodes, kg.src, kg.dst, kg.label_class, kg.term_ptr, kg.postings)
    g.set_label_weights(0.5, kg.avg_hops)
    g.set_debug(True)
    og = O.Graph(kg.n_nodes, kg.src, kg.dst, _oracle_act(kg))
    res = g.search_batch(qs.central, qs.marginal, qs.k, qs.depth)
    n_nonempty = 0
    for i, r in enumerate(res):
        ro = _oracle_run(og, kg.posting, qs.central[i], qs.marginal[i], qs.k, qs.depth)
        _cmp_results(r, ro)
        assert r.candidates == [(c.sc, c.v) for c in ro.candidates]
        n_nonempty += len(r.rpgs) > 0
    assert n_nonempty >= 20
    # single-query entry point agrees with the batch
    for i in range(5):
        _cmp_results(g.search(qs.central[i], qs.marginal[i], qs.k, qs.depth), res[i])


def test_search_mixed_term_counts_and_wide_rows(P):
    # T up to 8 per phase -> 64-bit H rows; batch mixes M = empty and |M| = 8
    rng = np.random.default_rng(91)
    V, src, dst, act, _ = random_instance(rng, 100, 400, deg=3.0, amax=4)
    post = [np.unique(rng.integers(0, V, int(rng.integers(1, 5)))).astype(np.uint32) for _ in range(20)]
    g = _dev_graph(P, V, src, dst, act, post)
    og = O.Graph(V, src, dst, act)
    Cs, Ms = [], []
    for i in range(24):
        nc = int(rng.integers(1, 9))
        nm = int(rng.choice([0, 1, 2, 5, 8]))
        tt = rng.choice(20, nc + nm, replace=True)
        Cs.append(tt[:nc].tolist())
        Ms.append(tt[nc:].tolist())
    res = g.search_batch(Cs, Ms, 4, 20)
    for i, r in enumerate(res):
        _cmp_results(r, _oracle_run(og, lambda t: post[t], Cs[i], Ms[i], 4, 20))


@pytest.mark.slow
def test_search_c2_sampled_queries(P):
    # full-size config 2 (1M nodes / 5M edges), the bench workload, in the bench's launch
    # configuration (one batch); exact comparison on a 12-query sample the oracle finishes
    kg = synth.make_kg(2)
    qs = synth.config_queries(kg, 2)
    g = P.Graph(kg.n_nodes, kg.src, kg.dst, kg.label_class, kg.term_ptr, kg.postings)
    g.set_label_weights(0.5, kg.avg_hops)
    w = O.fine_weights(kg.n_nodes, kg.src, kg.dst, kg.label_class)
    a = O.coarsen_all(w, 0.5, kg.avg_hops)
    assert (g.activation_levels() == a).all()
    og = O.Graph(kg.n_nodes, kg.src, kg.dst, a)
    res = g.search_batch(qs.central, qs.marginal, qs.k, qs.depth)
    for i in range(0, 200, 17):
        ro = _oracle_run(og, kg.posting, qs.central[i], qs.marginal[i], qs.k, qs.depth, want_matrices=False)
        _cmp_results(res[i], ro)
        assert res[i].stats["relax_marginal"] == ro.relax_m and res[i].stats["L_marginal"] == ro.Lm
    # full H parity for one query's central run
    H, blk, rel, L = g.hitting_levels(np.array(qs.central[0], np.uint32), 20, 1)
    Ho, bo, Lo, relo = O.phase(og, [kg.posting(t) for t in qs.central[0]], 20, 1)
    assert (H == Ho).all() and (blk == bo).all() and rel == relo


# ---------------------------------------------------------------- errors and edge cases
def test_error_codes(P):
    s, t, a = undirected_to_directed([[0, 1, 1], [1, 2, 1]])
    tp = np.array([0, 1, 2, 2], np.uint64)
    po = np.array([0, 2], np.uint32)
    g = P.Graph(3, s, t, None, tp, po)
    with pytest.raises(P.RikiError) as e:
        g.search([0], [], 1, 20)
    assert e.value.name == "RIKI_ENOWEIGHTS"
    g.set_activation_levels(a)
    for args, name in [(([], [1], 1, 20), "RIKI_EEMPTY_CENTRAL"), (([0], [2], 1, 20), "RIKI_EUNRESOLVED"),
                       (([0], [1], 1, 255), "RIKI_EDEPTH"), (([0], [1], 0, 20), "RIKI_EINVAL"),
                       (([7], [], 1, 20), "RIKI_EINVAL")]:
        with pytest.raises(P.RikiError) as e:
            g.search(*args)
        assert e.value.name == name, (args, e.value)
    with pytest.raises(P.RikiError):
        g.set_edge_weights(np.full(4, 1.5), 0.5, 4.0)
    with pytest.raises(P.RikiError):
        g.set_edge_weights(np.full(4, 0.5), 1.5, 4.0)
    # depth 0: only level-0 identification; nothing connects two different nodes
    r = g.search([0, 1], [], 1, 0)
    assert r.rpgs == []
    r = g.search([0], [], 2, 20)   # |C| = 1: keyword node itself, score 0
    assert [(x.central_node, x.sc) for x in r.rpgs] == [(0, 0)]


def test_empty_graph_edges(P):
    g = P.Graph(4, np.zeros(0, np.uint32), np.zeros(0, np.uint32), None, np.array([0, 2, 3], np.uint64),
                np.array([0, 3, 3], np.uint32))
    g.set_activation_levels(np.zeros(0, np.uint8))
    r = g.search([0, 1], [], 3, 20)
    assert [(x.central_node, x.sc) for x in r.rpgs] == [(3, 0)]


def test_device_batch_api(P):
    import torch
    kg = synth.make_kg(1)
    qs = synth.config_queries(kg, 1)
    g = P.Graph(kg.n_nodes, kg.src, kg.dst, kg.label_class, kg.term_ptr, kg.postings)
    g.set_label_weights(0.5, kg.avg_hops)
    cp, ct = P.Graph._csr(qs.central)
    mp, mt = P.Graph._csr(qs.marginal)
    d = [torch.from_numpy(x.astype(np.int64 if x.dtype == np.uint64 else np.int32)).cuda() for x in (cp, ct, mp, mt)]
    torch.cuda.synchronize()
    n = len(qs.central)
    g.search_batch_device(n, d[0].data_ptr(), d[1].data_ptr(), d[2].data_ptr(), d[3].data_ptr(), qs.k, qs.depth)
    got = g.fetch(n, [len(c) for c in qs.central], [len(m) for m in qs.marginal])
    ref = g.search_batch(qs.central, qs.marginal, qs.k, qs.depth)
    for a, b in zip(got, ref):
        _cmp_results(a, b)


@pytest.mark.parametrize("seed", range(6))
def test_direction_optimising_matches_push_and_oracle(P, seed):
    # hub-heavy graph: in-degree > 32 hubs exercise the warp-per-node pull path, dense
    # frontiers the thread-per-node path; push-only must agree bit for bit
    rng = np.random.default_rng(8100 + seed)
    V = 3000
    m = 9000
    hubs = rng.integers(0, V, 12)
    u = rng.integers(0, V, m)
    v = np.where(rng.random(m) < 0.4, hubs[rng.integers(0, 12, m)], rng.integers(0, V, m))
    v = np.where(u == v, (v + 1) % V, v)
    src = np.empty(2 * m, np.uint32); dst = np.empty(2 * m, np.uint32)
    src[0::2], dst[0::2] = u, v
    src[1::2], dst[1::2] = v, u
    act = rng.integers(0, 5, 2 * m).astype(np.uint8)
    post = [np.unique(rng.integers(0, V, int(rng.integers(1, 30)))).astype(np.uint32) for _ in range(8)]
    g = _dev_graph(P, V, src, dst, act, post)
    og = O.Graph(V, src, dst, act)
    for mode in (0, 1, 2):
        terms = np.arange(4, dtype=np.uint32)
        ref = O.phase(og, [post[t] for t in terms], 20, mode)
        for direction in (1, 0):
            g.set_direction(direction)
            H, blk, rel, L = g.hitting_levels(terms, 20, mode)
            assert (H == ref[0]).all() and (blk == ref[1]).all() and L == ref[2] and rel == ref[3]
    C, M = [0, 1], [2, 3]
    ro = _oracle_run(og, lambda t: post[t], C, M, 5, 20)
    for direction in (0, 1):
        g.set_direction(direction)
        _cmp_results(g.search(C, M, 5, 20), ro)


@pytest.mark.parametrize("seed", range(40))
def test_search_modes_marginal_heavy(P, seed):
    # |M| in {2, 3}: every PTC mode and early-termination mode against the oracle
    rng = np.random.default_rng(9100 + seed)
    V, src, dst, act, _ = random_instance(rng, 8, 40, deg=2.5, amax=3)
    post = [np.unique(rng.integers(0, V, int(rng.integers(1, 3)))).astype(np.uint32) for _ in range(8)]
    g = _dev_graph(P, V, src, dst, act, post)
    og = O.Graph(V, src, dst, act)
    nc, nm = int(rng.integers(1, 3)), int(rng.integers(2, 4))
    tt = rng.choice(8, nc + nm, replace=False)
    C, M = tt[:nc], tt[nc:]
    for ptc_mode in range(4):
        for early_term in range(3):
            kw = dict(ptc_mode=ptc_mode, early_term=early_term)
            _cmp_results(g.search(C, M, 3, 20, **kw), _oracle_run(og, lambda t: post[t], C, M, 3, 20, **kw))


@pytest.mark.slow
def test_search_c3_dbpedia_shaped_sampled(P):
    # config 3: 5M nodes / 20M directed edges, 3 central + 3 marginal, k = 20; the bench's
    # launch configuration: the whole 1k-query batch through the device path (it needs more
    # than 2^32 words of recovery arena, so it runs in chunks); 4 queries compared exactly,
    # spread over the chunks
    import torch
    kg = synth.make_kg(3)
    qs = synth.config_queries(kg, 3)
    nq = len(qs.central)
    g = P.Graph(kg.n_nodes, kg.src, kg.dst, kg.label_class, kg.term_ptr, kg.postings)
    g.set_label_weights(0.5, kg.avg_hops)
    g.set_batch_slots(min(nq, 1024))
    a = O.coarsen_all(O.fine_weights(kg.n_nodes, kg.src, kg.dst, kg.label_class), 0.5, kg.avg_hops)
    assert (g.activation_levels() == a).all()
    og = O.Graph(kg.n_nodes, kg.src, kg.dst, a)
    cp, ct = P.Graph._csr(qs.central)
    mp, mt = P.Graph._csr(qs.marginal)
    d = [torch.from_numpy(x.view(np.int64) if x.dtype == np.uint64 else x.view(np.int32)).cuda()
         for x in (cp, ct, mp, mt)]
    g.search_batch_device(nq, *(x.data_ptr() for x in d), qs.k, qs.depth)
    res = g.fetch(nq, [len(c) for c in qs.central], [len(m) for m in qs.marginal])
    for i in (0, 333, 666, 999):
        ro = _oracle_run(og, kg.posting, qs.central[i], qs.marginal[i], qs.k, qs.depth, want_matrices=False)
        _cmp_results(res[i], ro)
        assert res[i].stats["relax_central"] == ro.relax_c and res[i].stats["relax_marginal"] == ro.relax_m


def test_joint_traversal_c1_batch(P):
    # joint multi-query traversal (node-major H, union frontier) == oracle, query by query
    kg = synth.make_kg(1)
    qs = synth.config_queries(kg, 1)
    g = P.Graph(kg.n_nodes, kg.src, kg.dst, kg.label_class, kg.term_ptr, kg.postings)
    g.set_label_weights(0.5, kg.avg_hops)
    og = O.Graph(kg.n_nodes, kg.src, kg.dst, _oracle_act(kg))
    g.set_joint(True)
    res = g.search_batch(qs.central, qs.marginal, qs.k, qs.depth)
    for i, r in enumerate(res):
        ro = _oracle_run(og, kg.posting, qs.central[i], qs.marginal[i], qs.k, qs.depth)
        _cmp_results(r, ro)
        assert r.stats["relax_central"] == ro.relax_c and r.stats["relax_marginal"] == ro.relax_m
        assert r.stats["L_central"] == ro.Lc and r.stats["L_marginal"] == ro.Lm


@pytest.mark.parametrize("seed", range(6))
def test_joint_traversal_random_batches(P, seed):
    rng = np.random.default_rng(9900 + seed)
    V, src, dst, act, _ = random_instance(rng, 300, 2000, deg=3.0, amax=4)
    post = [np.unique(rng.integers(0, V, int(rng.integers(1, 6)))).astype(np.uint32) for _ in range(24)]
    g = _dev_graph(P, V, src, dst, act, post)
    g.set_debug(True)
    og = O.Graph(V, src, dst, act)
    nq = int(rng.choice([40, 64, 100]))
    Cs, Ms = [], []
    maxt = int(rng.choice([2, 4]))
    for _ in range(nq):
        nc = int(rng.integers(1, maxt + 1))
        nm = int(rng.integers(0, maxt + 1))
        tt = rng.choice(24, nc + nm, replace=False)
        Cs.append(tt[:nc].tolist())
        Ms.append(tt[nc:].tolist())
    k = int(rng.choice([1, 4]))
    g.set_joint(True)
    res = g.search_batch(Cs, Ms, k, 20)
    g.set_joint(False)
    ref = g.search_batch(Cs, Ms, k, 20)
    for i in range(nq):
        _cmp_results(res[i], ref[i])
        assert res[i].candidates == ref[i].candidates and res[i].stats == ref[i].stats
        if i % 7 == 0:
            ro = _oracle_run(og, lambda t: post[t], Cs[i], Ms[i], k, 20)
            _cmp_results(res[i], ro)
            assert res[i].stats["relax_central"] == ro.relax_c and res[i].stats["relax_marginal"] == ro.relax_m


@pytest.mark.slow
def test_joint_traversal_c2_sampled(P):
    kg = synth.make_kg(2)
    qs = synth.config_queries(kg, 2)
    g = P.Graph(kg.n_nodes, kg.src, kg.dst, kg.label_class, kg.term_ptr, kg.postings)
    g.set_label_weights(0.5, kg.avg_hops)
    g.set_joint(True)
    res = g.search_batch(qs.central, qs.marginal, qs.k, qs.depth)
    g.set_joint(False)
    ref = g.search_batch(qs.central, qs.marginal, qs.k, qs.depth)
    for i in range(len(res)):
        _cmp_results(res[i], ref[i])
        assert res[i].stats == ref[i].stats
    og = O.Graph(kg.n_nodes, kg.src, kg.dst, _oracle_act(kg))
    for i in (0, 99, 199):
        _cmp_results(res[i], _oracle_run(og, kg.posting, qs.central[i], qs.marginal[i], qs.k, qs.depth,
                                         want_matrices=False))
