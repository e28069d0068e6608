"""Pins for the CPU oracle (-m "not gpu").  Each test ties an oracle function to
something other than itself: values derived in SPEC/SURVEY from the paper's
equations, closed forms, textbook special cases, brute force, and an
independent event-driven evaluator (tests/brute.py)."""
import numpy as np
import pytest
from scipy.sparse import csr_matrix
from scipy.sparse.csgraph import shortest_path

import brute
import oracle as O
import synth
from fixtures import load_golden, random_instance, undirected_to_directed

INF = 0xFF


# ----------------------------------------------------------------- coarsening
def test_coarsen_worked_values():
    # SPEC S:142-144, derived from Eq. 1-3
    assert O.coarsen(0.5, 0.5, 4.0) == 4          # w = alpha -> Rounding(A)
    assert O.coarsen(0.0, 0.5, 4.0) == 0          # reward A
    assert O.coarsen(1.0, 0.5, 4.0) == 8          # penalty A
    assert O.coarsen(0.75, 0.5, 4.0) == 6         # 4 + 4*(0.25/0.5)
    assert O.coarsen(0.25, 0.5, 4.0) == 2         # consistency witness S:152


def test_bound_worked_values():
    # SPEC S:151-153 from Theorem boundEdgeWeight
    assert O.bound(2, 0.5, 4.0) == pytest.approx((0.1875, 0.3125))
    assert O.bound(4, 0.5, 4.0) == pytest.approx((0.4375, 0.5625))


def test_coarsen_bound_roundtrip_and_invariants():
    # SPEC acceptance 1: 1e4 random triples, w in bound(coarsen(w)); monotone; range.
    rng = np.random.default_rng(7)
    for _ in range(10000):
        w = float(rng.random())
        alpha = float(rng.choice([0.2, 0.5, 0.8]))
        A = float(rng.uniform(2, 6))
        a = O.coarsen(w, alpha, A)
        lo, hi = O.bound(a, alpha, A)
        assert lo - 1e-12 <= w < hi + 1e-12, (w, alpha, A, a, lo, hi)
        assert 0 <= a <= int(np.floor(2 * A + 0.5))
        # closed form of case 1: A - A(alpha-w)/alpha = A w / alpha (away from .5 ties)
        if w <= alpha:
            x = A * w / alpha
            if abs(x - np.floor(x) - 0.5) > 1e-9:
                assert a == int(np.floor(x + 0.5))
    ws = np.sort(rng.random(2000))
    a = O.coarsen_all(ws, 0.5, 3.87)
    assert (np.diff(a.astype(int)) >= 0).all()


def test_ln_count_correctly_rounded():
    # R31: P:193's log of an integer count is the fp64 value nearest to ln n.  Pinned by an
    # exact decimal evaluation (60 digits, then Python's correctly rounded str -> float), on
    # random integers and on integers where the C library's log is off by one ulp
    from decimal import Decimal, getcontext
    getcontext().prec = 60
    rng = np.random.default_rng(31)
    ns = [1, 2, 3, 10, 9170, 136837, 141614, 147674, 277862, 278555, 330034, 351497, 372772, 394915]
    ns += [int(x) for x in rng.integers(2, 1 << 32, 3000)]
    for n in ns:
        assert O.ln_count(n) == float(Decimal(n).ln()), n


def test_fine_weights_hand_fixtures():
    # lone edge -> log 2; 3 same-label out-edges into single-in targets -> log 4;
    # uniform graph -> all 0 (degenerate rescale, R2).
    # star v->a,v->b,v->c (label 0) + lone x->y (label 1); reverse edges class 2L+1.
    src = np.array([0, 1, 0, 2, 0, 3, 4, 5], np.uint32)
    dst = np.array([1, 0, 2, 0, 3, 0, 5, 4], np.uint32)
    cls = np.array([0, 1, 0, 1, 0, 1, 2, 3], np.uint32)
    w = O.fine_weights(6, src, dst, cls)
    # raw: star edges ln(3+1), their reverses ln(1+3), lone edges ln(1+1); min ln2, max ln4
    assert np.allclose(w, [1, 1, 1, 1, 1, 1, 0, 0])
    # mixed: a 2-edge fan (raw ln 3) sits halfway between ln2 and ln4 in log space? no:
    # (ln3 - ln2)/(ln4 - ln2) = log2(1.5)
    src2 = np.concatenate([src, np.array([6, 7, 6, 8], np.uint32)])
    dst2 = np.concatenate([dst, np.array([7, 6, 8, 6], np.uint32)])
    cls2 = np.concatenate([cls, np.array([4, 5, 4, 5], np.uint32)])
    w2 = O.fine_weights(9, src2, dst2, cls2)
    assert np.allclose(w2[8:], np.log2(1.5))
    u = O.fine_weights(2, np.array([0, 1], np.uint32), np.array([1, 0], np.uint32), np.array([0, 1], np.uint32))
    assert (u == 0).all()


def test_fine_weights_bruteforce_counts():
    rng = np.random.default_rng(3)
    V, E = 30, 200
    src = rng.integers(0, V, E).astype(np.uint32)
    dst = rng.integers(0, V, E).astype(np.uint32)
    cls = rng.integers(0, 4, E).astype(np.uint32)
    w = O.fine_weights(V, src, dst, cls)
    raw = np.array([np.log(np.sum((src == src[e]) & (cls == cls[e])) + np.sum((dst == dst[e]) & (cls == cls[e])))
                    for e in range(E)])
    ref = (raw - raw.min()) / (raw.max() - raw.min())
    assert np.allclose(w, ref, rtol=0, atol=1e-15)


# ----------------------------------------------------------------- path scoring
def test_path_score_examples_and_closed_form():
    assert O.path_score([]) == 0 and O.path_score([2, 1]) == 4 and O.path_score([1, 5]) == 6
    rng = np.random.default_rng(11)
    for _ in range(3000):
        seq = rng.integers(0, 10, int(rng.integers(0, 12))).tolist()
        assert O.path_score(seq) == brute.path_score_closed(seq)


def test_rpg_score_examples():
    assert O.rpg_score(0.5, 2, 4) == 3.0
    assert O.rpg_score(1.0, 2, 7) == 2.0 and O.rpg_score(0.0, 2, 7) == 7.0  # endpoints S:234
    assert O.rpg_score(0.3, 2, 2) == pytest.approx(2.0)


# ----------------------------------------------------------------- hitting levels (Alg. 1)
def test_known_answer_levels():
    d = load_golden("two_node.json")
    for case in d["cases"]:
        s, t, a = undirected_to_directed(case["undirected_edges"])
        g = O.Graph(case["nodes"], s, t, a)
        H, blk, L, _ = O.phase(g, [np.array(x, np.uint32) for x in case["terms"]], case["depth"], 0)
        assert H.tolist() == case["expect_H"]


def _bfs_levels(V, src, dst, sources):
    A = csr_matrix((np.ones(len(src)), (src.astype(np.int64), dst.astype(np.int64))), shape=(V, V))
    d = shortest_path(A, unweighted=True, directed=True, indices=np.asarray(sources, np.int64))
    return d.min(axis=0) if d.ndim == 2 else d


@pytest.mark.parametrize("seed", range(40))
def test_levels_special_cases_and_dijkstra(seed):
    rng = np.random.default_rng(100 + seed)
    V, src, dst, act, terms = random_instance(rng, 5, 40, T_hi=3)
    D = int(rng.choice([3, 5, 8, 20]))
    # textbook case: all a = 0, no blocking -> multi-source BFS hops (capped at D)
    g0 = O.Graph(V, src, dst, np.zeros_like(act))
    H0, _, _, _ = O.phase(g0, terms, D, 0)
    for j, t in enumerate(terms):
        bfs = _bfs_levels(V, src, dst, t)
        ref = np.where(np.isfinite(bfs) & (bfs <= D), bfs, INF).astype(np.int64)
        assert (H0[:, j].astype(np.int64) == ref).all()
    # a == c everywhere -> h = c + hops for hops >= 1
    c = int(rng.integers(1, 4))
    gc = O.Graph(V, src, dst, np.full_like(act, c))
    Hc, _, _, _ = O.phase(gc, terms, 40, 0)
    for j, t in enumerate(terms):
        bfs = _bfs_levels(V, src, dst, t)
        ref = np.where(np.isfinite(bfs), np.where(bfs >= 1, bfs + c, 0), INF)
        assert (Hc[:, j].astype(np.int64) == ref.astype(np.int64)).all()
    # general activations, no blocking: label-correcting Dijkstra on Def. pathScoring
    g = O.Graph(V, src, dst, act)
    H, _, _, _ = O.phase(g, terms, D, 0)
    for j, t in enumerate(terms):
        dj = brute.dijkstra_levels(V, src, dst, act, t)
        ref = np.where(dj <= D, dj, INF)
        assert (H[:, j].astype(np.int64) == ref).all()
        # north-star invariant: finite h >= unweighted BFS distance
        bfs = _bfs_levels(V, src, dst, t)
        fin = H[:, j] != INF
        assert (H[fin, j] >= bfs[fin]).all()
    # with central blocking the invariant still holds
    Hb, _, _, _ = O.phase(g, terms, D, 1)
    for j, t in enumerate(terms):
        bfs = _bfs_levels(V, src, dst, t)
        fin = Hb[:, j] != INF
        assert (Hb[fin, j] >= bfs[fin]).all()


@pytest.mark.parametrize("seed", range(12))
def test_levels_bruteforce_paths(seed):
    rng = np.random.default_rng(500 + seed)
    V, src, dst, act, terms = random_instance(rng, 4, 9, deg=2.0, T_hi=2)
    g = O.Graph(V, src, dst, act)
    H, _, _, _ = O.phase(g, terms, 40, 0)
    for j, t in enumerate(terms):
        bp = brute.brute_levels(V, src, dst, act, t)
        assert (H[:, j].astype(np.int64) == bp).all()


@pytest.mark.parametrize("seed", range(60))
def test_levels_match_event_driven_with_blocking(seed):
    # O1 (literal level-synchronous Alg. 1 with CF) == O2 (event buckets, closed-form blocking)
    rng = np.random.default_rng(900 + seed)
    V, src, dst, act, terms = random_instance(rng, 5, 40, T_hi=4)
    D = int(rng.choice([3, 5, 8, 20]))
    g = O.Graph(V, src, dst, act)
    for mode in (0, 1, 2):
        H, blk, L, _ = O.phase(g, terms, D, mode)
        blocking = mode == 1 or (mode == 2 and len(terms) >= 2)
        H2 = brute.o2_levels(V, src, dst, act, terms, D, blocking)
        assert (H.astype(np.int64) == H2).all(), mode
        # R10 closed form: block = max row if complete, else inf (only when blocking)
        comp = (H != INF).all(axis=1)
        ref = np.where(comp, H.max(axis=1), INF) if blocking else np.full(V, INF)
        assert (blk.astype(np.int64) == ref.astype(np.int64)).all()


@pytest.mark.parametrize("seed", range(60))
def test_phase_relaxations_and_end_level_match_event_counts(seed):
    # SURVEY §8(d) relaxation count R (the GTEPS numerator) and the terminating level of a raw
    # run, pinned by O2's event count per bucket and an independent frontier-emptiness rule
    # (tests/brute.py::o2_phase); a mistake such as counting L <= L_end, ignoring blocking or
    # stopping one level late fails here
    rng = np.random.default_rng(900 + seed)
    V, src, dst, act, terms = random_instance(rng, 5, 40, T_hi=4)
    D = int(rng.choice([3, 5, 8, 20]))
    g = O.Graph(V, src, dst, act)
    for mode in (0, 1, 2):
        H, blk, L, rel = O.phase(g, terms, D, mode)
        blocking = mode == 1 or (mode == 2 and len(terms) >= 2)
        H2, L2, R2 = brute.o2_phase(V, src, dst, act, terms, D, blocking)
        assert (H.astype(np.int64) == H2).all()
        assert L == L2, (mode, L, L2)
        assert rel == R2, (mode, rel, R2)


@pytest.mark.parametrize("seed", range(40))
def test_search_relaxations_match_event_counts(seed):
    # the search's per-run relaxation counts (bench GTEPS numerator) against O2's events below
    # each run's terminating level; the central terminating level itself against its definition
    # ("at least w CGs", R8 depth, empty frontier)
    rng = np.random.default_rng(2000 + seed)
    V, src, dst, act, _ = random_instance(rng, 6, 18, deg=2.2, amax=4)
    nc, nm = int(rng.integers(1, 4)), int(rng.integers(1, 4))
    terms = [np.unique(rng.integers(0, V, int(rng.integers(1, 4)))).astype(np.uint32) for _ in range(nc + nm)]
    C, M = terms[:nc], terms[nc:]
    k = int(rng.choice([1, 3, 5]))
    D = int(rng.choice([3, 6, 20]))
    r = O.search(O.Graph(V, src, dst, act), C, M, k, D)
    ev = [0] * D
    Hc = brute.o2_levels(V, src, dst, act, C, D, True, ev)
    _, Lend, _ = brute.o2_phase(V, src, dst, act, C, D, True)
    mx = np.where((Hc != INF).all(axis=1), Hc.max(axis=1), INF)
    Lw = next((L for L in range(D + 1) if (mx <= L).sum() >= k), D)
    assert r.Lc == min(Lw, Lend)
    assert r.relax_c == sum(ev[:r.Lc])
    if r.Lm >= 0:
        evm = [0] * D
        brute.o2_levels(V, src, dst, act, M, D, nm >= 2, evm)
        assert r.relax_m == sum(evm[:r.Lm])


@pytest.mark.parametrize("seed", range(20))
def test_levels_depth_truncation_and_permutation(seed):
    rng = np.random.default_rng(1300 + seed)
    V, src, dst, act, terms = random_instance(rng, 5, 40, T_hi=3)
    g = O.Graph(V, src, dst, act)
    for mode in (0, 1):
        Hd, _, _, _ = O.phase(g, terms, 4, mode)
        Hf, _, _, _ = O.phase(g, terms, 30, mode)
        assert (Hd == np.where(Hf <= 4, Hf, INF)).all()
        perm = rng.permutation(len(src))
        gp = O.Graph(V, src[perm], dst[perm], act[perm])
        Hp, bp, _, _ = O.phase(gp, terms, 30, mode)
        assert (Hp == Hf).all()


def test_alpha_monotonicity():
    # smaller alpha -> pointwise larger-or-equal a -> pointwise larger-or-equal H (no blocking)
    rng = np.random.default_rng(5)
    for _ in range(30):
        V, src, dst, _, terms = random_instance(rng, 5, 30)
        w = rng.random(len(src))
        a3 = O.coarsen_all(w, 0.3, 3.87)
        a7 = O.coarsen_all(w, 0.7, 3.87)
        assert (a3 >= a7).all()
        H3, _, _, _ = O.phase(O.Graph(V, src, dst, a3), terms, 30, 0)
        H7, _, _, _ = O.phase(O.Graph(V, src, dst, a7), terms, 30, 0)
        assert (H3 >= H7).all()


# ----------------------------------------------------------------- end-to-end fixtures
def _run_fixture(name, **kw):
    d = load_golden(name)
    s, t, a = undirected_to_directed(d["undirected_edges"])
    g = O.Graph(d["nodes"], s, t, a)
    C = [np.array(x, np.uint32) for x in d["central"]]
    M = [np.array(x, np.uint32) for x in d["marginal"]]
    r = O.search(g, C, M, d["k"], d["depth"], gamma=d["gamma"], **kw)
    return d, s, t, r


@pytest.mark.parametrize("name", ["five_node.json", "diamond.json", "r16_blocked_relay.json",
                                  "ptc_fail_m2.json", "ptc_fail_m3.json", "ptc_pass_vc_marginal.json"])
def test_golden_end_to_end(name):
    d, s, t, r = _run_fixture(name)
    assert len(r.rpgs) == len(d["expect"])
    for got, exp in zip(r.rpgs, d["expect"]):
        assert got.central_node == exp["central_node"]
        assert got.sc == exp["sc"] and got.sm == exp["sm"] and got.score == exp["score"]
        assert got.nodes.tolist() == exp["nodes"]
        de = sorted((int(s[e]), int(t[e])) for e in got.edge_ids)
        assert de == sorted(tuple(x) for x in exp["directed_edges"])
    if "expect_ptc_fail" in d:
        assert r.n_ptc_fail == d["expect_ptc_fail"]


def _check_rpgs(rpgs, expect, s, t):
    assert len(rpgs) == len(expect), (len(rpgs), len(expect))
    for got, exp in zip(rpgs, expect):
        assert (got.central_node, got.sc, got.sm, got.score) == (exp["central_node"], exp["sc"], exp["sm"],
                                                                 exp["score"])
        assert int(got.ptc) == exp["ptc"]
        assert got.nodes.tolist() == exp["nodes"]
        assert sorted((int(s[e]), int(t[e])) for e in got.edge_ids) == sorted(tuple(x) for x in exp["directed_edges"])


@pytest.mark.parametrize("name", ["ptc_gm_only_r20i.json", "ptc_single_marginal_node.json",
                                  "early_term_literal_gamma1.json"])
def test_golden_mode_fixtures(name):
    # hand-derived fixtures for the option paths: ptc_mode 2 (G^m-only PTC, R20 case (i)),
    # R19' ("at least two different marginal keyword nodes") and the paper-literal early
    # termination (early_term 1) where it differs from the exact bound R21
    d = load_golden(name)
    s, t, a = undirected_to_directed(d["undirected_edges"])
    g = O.Graph(d["nodes"], s, t, a)
    C = [np.array(x, np.uint32) for x in d["central"]]
    M = [np.array(x, np.uint32) for x in d["marginal"]]
    for run in d["runs"]:
        r = O.search(g, C, M, d["k"], d["depth"], gamma=d["gamma"], **run["params"])
        _check_rpgs(r.rpgs, run["expect"], s, t)
        if "expect_ptc_fail" in run:
            assert r.n_ptc_fail == run["expect_ptc_fail"], run["params"]
        if "expect_L_marginal" in run:
            assert r.Lm == run["expect_L_marginal"], run["params"]


@pytest.mark.parametrize("seed", range(60))
def test_literal_early_termination_exact_below_gamma_one(seed):
    # early_term 1 (P:375-381 literal) for 0 <= gamma < 1: S^r(kth) <= g*min S^c + (1-g)*S^m(kth)
    # reduces to S^c(kth) <= min S^c(unattached), and every unattached CG has S^m >= l+1 > S^m(kth),
    # so it never changes the answer: it must equal the plain-definition (exhaustive) form
    rng = np.random.default_rng(7700 + seed)
    V, src, dst, act, _ = random_instance(rng, 8, 20, deg=2.5, amax=3)
    nc, nm = int(rng.integers(1, 3)), int(rng.integers(1, 4))
    terms = [np.unique(rng.integers(0, V, int(rng.integers(1, 3)))).astype(np.uint32) for _ in range(nc + nm)]
    C, M = terms[:nc], terms[nc:]
    k = int(rng.choice([1, 3, 5]))
    gamma = float(rng.choice([0.0, 0.25, 0.5, 0.9]))
    r = O.search(O.Graph(V, src, dst, act), C, M, k, 20, gamma=gamma, early_term=1)
    ref, _ = brute.search_plain(V, src, dst, act, C, M, k, 20, gamma=gamma)
    assert [(x.score, x.sc, x.central_node, x.sm, x.nodes.tolist(), sorted(int(e) for e in x.edge_ids))
            for x in r.rpgs] == [(x[0], x[1], x[2], x[3], x[4], x[5]) for x in ref]


def test_ptc_modes_on_vc_marginal():
    # exclusive form rejects what the inclusive reading (R19) accepts
    _, _, _, r3 = _run_fixture("ptc_pass_vc_marginal.json", ptc_mode=3)
    assert len(r3.rpgs) == 0
    # flag-only keeps the PTC failure, flagged
    _, _, _, r1 = _run_fixture("ptc_fail_m2.json", ptc_mode=1)
    assert len(r1.rpgs) == 1 and r1.rpgs[0].ptc == 0


# ----------------------------------------------------------------- whole search vs plain definition
def _random_query(rng, V, src, dst, act):
    nc = int(rng.integers(1, 4))
    nm = int(rng.integers(0, 4))
    terms = [np.unique(rng.integers(0, V, int(rng.integers(1, 4)))).astype(np.uint32) for _ in range(nc + nm)]
    return terms[:nc], terms[nc:]


@pytest.mark.parametrize("seed", range(80))
def test_search_matches_plain_definition(seed):
    # early-terminated O1 == exhaustive plain-definition form built from
    # O2 + path enumeration + brute PTC (tests/brute.py)
    rng = np.random.default_rng(2000 + seed)
    V, src, dst, act, _ = random_instance(rng, 6, 18, deg=2.2, amax=4)
    C, M = _random_query(rng, V, src, dst, act)
    k = int(rng.choice([1, 3, 5]))
    D = int(rng.choice([3, 6, 20]))
    g = O.Graph(V, src, dst, act)
    r = O.search(g, C, M, k, D)
    ref, cands = brute.search_plain(V, src, dst, act, C, M, k, D)
    assert [(c.sc, c.v) for c in r.candidates] == cands
    got = [(x.score, x.sc, x.central_node, x.sm, x.nodes.tolist(), sorted(int(e) for e in x.edge_ids))
           for x in r.rpgs]
    exp = [(x[0], x[1], x[2], x[3], x[4], x[5]) for x in ref]
    assert got == exp
    # exhaustive mode gives the same answer (early termination must not change it)
    r2 = O.search(g, C, M, k, D, early_term=2)
    assert [(x.score, x.central_node, x.edge_ids.tolist()) for x in r2.rpgs] == \
           [(x.score, x.central_node, x.edge_ids.tolist()) for x in r.rpgs]


@pytest.mark.parametrize("seed", range(10))
def test_search_degenerate_cases(seed):
    rng = np.random.default_rng(4000 + seed)
    V, src, dst, act, _ = random_instance(rng, 8, 30, amax=4)
    g = O.Graph(V, src, dst, act)
    t0 = np.unique(rng.integers(0, V, 4)).astype(np.uint32)
    # |C| = 1: every central keyword node is a score-0 CG at level 0
    r = O.search(g, [t0], [], 2, 20)
    assert [(c.sc, c.v) for c in r.candidates] == [(0, int(v)) for v in t0]
    assert r.Lc == 0
    # M = empty: top-k CGs by (S^c, v), S^r = S^c
    t1 = np.unique(rng.integers(0, V, 3)).astype(np.uint32)
    r = O.search(g, [t0, t1], [], 3, 20)
    exp = sorted((c.sc, c.v) for c in r.candidates)[:3]
    assert [(x.sc, x.central_node) for x in r.rpgs] == exp
    assert all(x.score == x.sc for x in r.rpgs)
    # level-score law: identified CG scores never exceed the terminating level
    assert all(c.sc <= r.Lc for c in r.candidates)


@pytest.mark.parametrize("seed", range(150))
def test_search_plain_definition_marginal_heavy(seed):
    # |M| in {2,3}, low activations: exercises the stop rule, attach and PTC failures (R20)
    rng = np.random.default_rng(7000 + seed)
    V, src, dst, act, _ = random_instance(rng, 8, 20, deg=2.5, amax=3)
    nc = int(rng.integers(1, 3))
    nm = int(rng.integers(2, 4))
    terms = [np.unique(rng.integers(0, V, int(rng.integers(1, 3)))).astype(np.uint32) for _ in range(nc + nm)]
    C, M = terms[:nc], terms[nc:]
    k = int(rng.choice([1, 3, 5]))
    r = O.search(O.Graph(V, src, dst, act), C, M, k, 20)
    ref, _ = brute.search_plain(V, src, dst, act, C, M, k, 20)
    got = [(x.score, x.sc, x.central_node, x.sm, x.nodes.tolist(), sorted(int(e) for e in x.edge_ids))
           for x in r.rpgs]
    assert got == [(x[0], x[1], x[2], x[3], x[4], x[5]) for x in ref]


# ----------------------------------------------------------------- weight-sum tie-break (R29)
def _tie_fixture():
    d = load_golden("tie_break_weight_sum.json")
    e = d["directed_edges"]
    src = np.array([x[0] for x in e], np.uint32)
    dst = np.array([x[1] for x in e], np.uint32)
    wf = np.array([x[2] for x in e], np.float64)
    act = np.full(len(e), d["activation"], np.uint8)
    return d, src, dst, wf, act


def test_tie_break_golden_fixture():
    d, src, dst, wf, act = _tie_fixture()
    g = O.Graph(d["nodes"], src, dst, act)
    C = [np.array(x, np.uint32) for x in d["central"]]
    for case in d["cases"]:
        M = [np.array(x, np.uint32) for x in d["marginal"]] if case["marginal"] else []
        r = O.search(g, C, M, case["k"], d["depth"], gamma=d["gamma"], tie_break=case["tie_break"], wfine=wf,
                     beam_w=case.get("beam_w", 0), beam_mode=case.get("beam_mode", 0))
        assert [x.central_node for x in r.rpgs] == case["expect"], case
        for x, ws in zip(r.rpgs, case.get("wsum", [])):
            assert abs(x.wsum / 2.0 ** 32 - ws) < 1e-8, (case, x.wsum)
        for x, ed in zip(r.rpgs, case.get("edges", [])):
            assert x.edge_ids.tolist() == ed


def test_tie_break_exact_fixed_point():
    # R29: W is exact (integer units of 2^-32), so it does not depend on the summation order
    from fractions import Fraction
    for w in (0.0, 1.0, 0.5, 0.1, 0.3, 1 / 3, 2 ** -33, 1 - 2 ** -40):
        q = Fraction(w) * (1 << 32) + Fraction(1, 2)
        assert brute.weight_sum([0], [w]) == q.numerator // q.denominator
    assert brute.weight_sum([0, 0, 1], [0.25, 0.5]) == (1 << 30) + (1 << 31)  # distinct edges only


@pytest.mark.parametrize("seed", range(60))
def test_tie_break_matches_plain_definition(seed):
    # weights from a coarse grid (k/8) so equal-score results often tie on W too (then v decides)
    rng = np.random.default_rng(7700 + seed)
    V, src, dst, act, _ = random_instance(rng, 6, 16, deg=2.4, amax=2)
    wf = rng.integers(0, 9, len(src)) / 8.0
    C, M = _random_query(rng, V, src, dst, act)
    k = int(rng.choice([1, 2, 3, 5]))
    g = O.Graph(V, src, dst, act)
    r = O.search(g, C, M, k, 20, tie_break=1, wfine=wf)
    ref, _ = brute.search_plain(V, src, dst, act, C, M, k, 20, wfine=wf)
    got = [(x.score, x.sc, x.central_node, sorted(int(e) for e in x.edge_ids)) for x in r.rpgs]
    assert got == [(x[0], x[1], x[2], x[5]) for x in ref]
    assert [x.wsum for x in r.rpgs] == [brute.weight_sum(x[5], wf) for x in ref]
    r2 = O.search(g, C, M, k, 20, tie_break=1, wfine=wf, early_term=2)
    assert [(x.central_node, x.wsum) for x in r2.rpgs] == [(x.central_node, x.wsum) for x in r.rpgs]


@pytest.mark.parametrize("seed", range(30))
def test_tie_break_beam_truncation(seed):
    # beam_mode 1 + tie-break keeps the w smallest (S^c, W(CG), v) of the tie-kept candidate set
    rng = np.random.default_rng(7900 + seed)
    V, src, dst, act, _ = random_instance(rng, 6, 18, deg=2.4, amax=2)
    wf = rng.integers(0, 9, len(src)) / 8.0
    C, M = _random_query(rng, V, src, dst, act)
    g = O.Graph(V, src, dst, act)
    bw = int(rng.integers(1, 4))
    full = O.search(g, C, M, 1, 20, beam_w=bw, early_term=2)
    keys = sorted((c.sc, brute.weight_sum(c.cg_edges, wf), c.v) for c in full.candidates)[:bw]
    r = O.search(g, C, M, 1, 20, beam_w=bw, beam_mode=1, tie_break=1, wfine=wf, early_term=2)
    assert [(c.sc, c.v) for c in r.candidates] == sorted((sc, v) for sc, _, v in keys)


def test_oracle_is_reentrant_across_threads():
    # bench.py's cpu_baseline runs one oracle query per host thread: results must not depend on it
    from concurrent.futures import ThreadPoolExecutor
    kg = synth.make_kg(1)
    qs = synth.config_queries(kg, 1)
    og = O.Graph(kg.n_nodes, kg.src, kg.dst, O.coarsen_all(O.fine_weights(kg.n_nodes, kg.src, kg.dst,
                                                                          kg.label_class), 0.5, kg.avg_hops))

    def one(i):
        r = O.search(og, [kg.posting(t) for t in qs.central[i]], [kg.posting(t) for t in qs.marginal[i]], qs.k,
                     qs.depth, want_matrices=False, want_candidates=False)
        return [(x.central_node, x.score, x.edge_ids.tolist()) for x in r.rpgs]

    seq = [one(i) for i in range(len(qs.central))]
    with ThreadPoolExecutor(8) as ex:
        par = list(ex.map(one, range(len(qs.central))))
    assert par == seq


# ----------------------------------------------------------------- Abar by sampled pairs (R30)
def _bfs_brute(V, src, dst, s):
    from collections import deque
    adj = [[] for _ in range(V)]
    for a, b in zip(src, dst):
        adj[int(a)].append(int(b))
    d = [None] * V
    d[s] = 0
    q = deque([s])
    while q:
        u = q.popleft()
        for w in adj[u]:
            if d[w] is None:
                d[w] = d[u] + 1
                q.append(w)
    return d


def test_sample_avg_hops_hand_fixtures():
    # path 0-1-2-3-4 (bidirected) plus a one-way edge 5 -> 0
    und = [(0, 1), (1, 2), (2, 3), (3, 4)]
    src = [a for a, b in und] + [b for a, b in und] + [5]
    dst = [b for a, b in und] + [a for a, b in und] + [0]
    m, sd, n, d = O.sample_avg_hops(6, src, dst, [0, 1, 2, 5, 0], [4, 3, 2, 4, 5])
    assert d.tolist() == [4, 2, 0, 5, O.HOP_INF]  # 0 cannot reach 5 (one-way edge)
    assert n == 4 and m == 11 / 4
    assert abs(sd - np.std([4, 2, 0, 5], ddof=1)) < 1e-15
    m, sd, n, d = O.sample_avg_hops(6, src, dst, [0, 1], [4, 3], max_hops=3)
    assert d.tolist() == [O.HOP_INF, 2] and n == 1 and m == 2.0 and np.isnan(sd)


@pytest.mark.parametrize("seed", range(20))
def test_sample_avg_hops_matches_brute_bfs(seed):
    import statistics
    rng = np.random.default_rng(8800 + seed)
    V, src, dst, _, _ = random_instance(rng, 5, 60, deg=float(rng.choice([1.0, 2.0, 3.0])))
    if seed % 3 == 0:  # some one-way edges
        keep = rng.random(len(src)) < 0.8
        src, dst = src[keep], dst[keep]
    ps = rng.integers(0, V, 40)
    pt = rng.integers(0, V, 40)
    m, sd, n, d = O.sample_avg_hops(V, src, dst, ps, pt)
    exp = []
    for s_, t_ in zip(ps, pt):
        x = _bfs_brute(V, src, dst, int(s_))[int(t_)]
        exp.append(O.HOP_INF if x is None else x)
    assert d.tolist() == exp
    ok = [x for x in exp if x != O.HOP_INF]
    assert n == len(ok)
    if len(ok) >= 1:
        assert abs(m - statistics.fmean(ok)) <= 1e-12 * max(1.0, m)
    if len(ok) >= 2:
        assert abs(sd - statistics.stdev(ok)) <= 1e-12 * max(1.0, sd)
