"""Independent slow checkers used to PIN the oracle (test-only, tiny inputs).

Nothing here calls oracle/ or the CUDA path.  Each function re-derives a
quantity from the paper's definitions by a different route than the oracle's
level-synchronous transcription of Alg. 1 / Alg. 2:

* ``path_score_closed``  closed form of Def. pathScoring:
  F([a_1..a_m]) = max(m, max_j (a_j + m - j + 1)).
* ``dijkstra_levels``    label-correcting best-first search under s' = max(s, a) + 1
  (Def. distKeyword2Node; valid since s' > s).
* ``brute_levels``       min over enumerated simple paths (tiny graphs).
* ``o2_levels``          event-driven bucket evaluator with blocking by the closed
  form of R10 (no frontier, no retention, no stored block array).
* ``sp_edges_brute``     union of prefix-optimal, realizable min-score simple paths
  (R27 + R16) by path enumeration.
* ``ptc_brute``          Def. RPG PTC by enumerating simple paths between
  marginal keyword nodes of the RPG and testing whether they avoid V_C.
* ``search_plain``       the plain-definition form of the whole search (SURVEY
  §8(c)): candidates from O2, CGs/RPGs from path enumeration, exhaustive
  marginal run, PTC, sort, take k.
"""
from __future__ import annotations

import heapq
from collections import defaultdict

import numpy as np

INF = 0xFF


def path_score_closed(seq):
    m = len(seq)
    if m == 0:
        return 0
    return max(m, max(a + m - j for j, a in enumerate(seq, start=1)) + 1)


def _adj(V, src, dst):
    out = [[] for _ in range(V)]
    inn = [[] for _ in range(V)]
    for e, (u, v) in enumerate(zip(src.tolist(), dst.tolist())):
        out[u].append(e)
        inn[v].append(e)
    return out, inn


def dijkstra_levels(V, src, dst, act, sources, cap=254):
    dist = [INF] * V
    pq = []
    for s in sources:
        if dist[s] != 0:
            dist[s] = 0
            heapq.heappush(pq, (0, s))
    out, _ = _adj(V, np.asarray(src), np.asarray(dst))
    while pq:
        d, u = heapq.heappop(pq)
        if d > dist[u]:
            continue
        for e in out[u]:
            nd = max(d, int(act[e])) + 1
            if nd <= cap and nd < dist[int(dst[e])]:
                dist[int(dst[e])] = nd
                heapq.heappush(pq, (nd, int(dst[e])))
    return np.array(dist, np.int64)


def brute_levels(V, src, dst, act, sources, max_edges=12):
    """min over simple paths (<= max_edges edges) of Def. pathScoring."""
    out, _ = _adj(V, np.asarray(src), np.asarray(dst))
    best = [INF] * V
    srcset = set(int(s) for s in sources)

    def dfs(u, score, depth, onpath):
        if score < best[u]:
            best[u] = score
        if depth == max_edges:
            return
        for e in out[u]:
            n = int(dst[e])
            if n in onpath:
                continue
            onpath.add(n)
            dfs(n, max(score, int(act[e])) + 1, depth + 1, onpath)
            onpath.discard(n)

    for s in srcset:
        dfs(s, 0, 0, {s})
    return np.array(best, np.int64)


def o2_levels(V, src, dst, act, terms, depth, blocking, events=None):
    """Event-driven evaluator.  At level L every settled (f, j) with key
    max(h_fj, a_e) == L relaxes e unless f is blocked at L; f is blocked at L iff
    blocking and its row is complete with max <= L (R10 closed form).
    Returns H (V x T, INF = 255).  ``events`` (a list of >= depth zeros), when given,
    receives the number of relaxation events processed in each bucket L."""
    T = len(terms)
    H = np.full((V, T), INF, np.int64)
    for j, t in enumerate(terms):
        for v in t:
            H[int(v), j] = 0
    out, _ = _adj(V, np.asarray(src), np.asarray(dst))
    act = np.asarray(act, np.int64)

    def blocked(f, L):
        return blocking and (H[f] != INF).all() and H[f].max() <= L

    for L in range(depth):
        updates = []
        for f in range(V):
            if blocked(f, L):
                continue
            for j in range(T):
                h = H[f, j]
                if h == INF or h > L:
                    continue
                for e in out[f]:
                    if max(h, act[e]) != L:
                        continue
                    if events is not None:
                        events[L] += 1
                    n = int(dst[e])
                    if H[n, j] == INF:
                        updates.append((n, j))
        for n, j in updates:
            H[n, j] = L + 1
    return H


def o2_phase(V, src, dst, act, terms, depth, blocking):
    """O2 extended with the two quantities the oracle's phase also reports, each derived from
    the paper's definitions by its own route (no frontier array, no re-scans):

    * L_end -- the first level l with an empty frontier, or ``depth``.  Alg. 1 keeps F_f = 1
      while f is unblocked and some out-edge has a_fn > l (lines 9-11), and sets
      F_n = 1 when n is first reached (line 17), so by induction f is in the frontier Phi_l
      (l >= 1) iff some column of f was reached at exactly l, or (f was reached before l,
      max_e a_e >= l and f was not blocked at l - 1).  Seeds form Phi_0.
    * R -- SURVEY §8(d)'s relaxation count, as the number of events the bucket queue
      processes in buckets L < L_end: (f, j, e) with key max(h_fj, a_e) = L and f not blocked
      at L (R10 closed form, tested while H holds only the final values <= L), counted whether
      or not the event reaches a new cell.

    Returns (H, L_end, R)."""
    events = [0] * max(depth, 1)
    H = o2_levels(V, src, dst, act, terms, depth, blocking, events)
    T = len(terms)
    out, _ = _adj(V, np.asarray(src), np.asarray(dst))
    act = np.asarray(act, np.int64)
    fin = H != INF
    comp = fin.all(axis=1)
    blk = np.where(comp, H.max(axis=1), INF) if blocking and T > 0 else np.full(V, INF)
    h0 = np.where(fin.any(axis=1), np.where(fin, H, INF).min(axis=1), INF)
    amax = np.array([max((int(act[e]) for e in out[f]), default=-1) for f in range(V)])

    def frontier_nonempty(l):
        if l == 0:
            return bool((h0 == 0).any())
        for f in range(V):
            if (H[f] == l).any():
                return True
            if h0[f] != INF and h0[f] <= l - 1 and amax[f] >= l and blk[f] > l - 1:
                return True
        return False

    L_end = depth
    for l in range(depth + 1):
        if not frontier_nonempty(l):
            L_end = l
            break
    R = sum(events[:L_end])
    return H, L_end, R


def enumerate_min_paths(V, src, dst, act, H, j, blockarr, targets, max_edges=14):
    """Union of edges over simple paths ending at a node in ``targets`` that start at a
    keyword node of column j (h = 0) and are (1) min-score: F = h[target], (2)
    prefix-optimal: F(prefix ending at x) = h[x] for every x, (3) realizable: every
    relay x forwards at level max(F_x, a) < block[x].  Paths are searched backwards
    from each target, so all simple paths are covered."""
    _, inn = _adj(V, np.asarray(src), np.asarray(dst))
    edges = set()
    nodes = set()

    # forward-check a full path (list of edge ids from source to target)
    def ok(path_edges, target):
        if not path_edges:
            return True
        s = 0
        first = int(src[path_edges[0]])
        if H[first, j] != 0:
            return False
        x = first
        for e in path_edges:
            L = max(s, int(act[e]))
            if L >= blockarr[x]:
                return False
            s = L + 1
            x = int(dst[e])
            if s != H[x, j]:
                return False
        return x == target and s == H[target, j]

    def back(x, path_rev, onpath, target):
        # path_rev: edges from x to target, reversed order
        if H[x, j] == 0:
            p = list(reversed(path_rev))
            if ok(p, target):
                for e in p:
                    edges.add(e)
                    nodes.add(int(src[e]))
                    nodes.add(int(dst[e]))
            # keyword nodes end paths (Alg. 2 line 10: no continuation through h = 0)
            return
        if len(path_rev) >= max_edges:
            return
        for e in inn[x]:
            n = int(src[e])
            if n in onpath or H[n, j] == INF:
                continue
            onpath.add(n)
            back(n, path_rev + [e], onpath, target)
            onpath.discard(n)

    for t in targets:
        if H[t, j] == INF:
            continue
        nodes.add(int(t))
        back(int(t), [], {int(t)}, int(t))
    return edges, nodes


def ptc_brute(V, src, dst, nodes, edges, vc, Hm, n_marg, max_len=30):
    """P:145 'There exists at least two different marginal keyword nodes in an RPG such
    that all their simple path connections (regardless of edge directions) must pass
    through nodes in V_C' -- endpoint-inclusive reading R19: a path whose endpoint is in
    V_C passes through V_C.  Pairs with no connection at all inside the RPG qualify
    vacuously (their connections all pass through V_C)."""
    if n_marg == 1:
        return True
    X = [v for v in sorted(nodes) if (Hm[v] == 0).any()]
    vcs = set(int(x) for x in vc)
    und = defaultdict(set)
    for e in edges:
        a, b = int(src[e]), int(dst[e])
        und[a].add(b)
        und[b].add(a)

    def has_avoiding_path(x1, x2):
        # DFS over simple paths that avoid V_C entirely (endpoints included)
        if x1 in vcs or x2 in vcs:
            return False
        stack = [x1]
        seen = {x1}
        while stack:
            u = stack.pop()
            if u == x2:
                return True
            for w in und[u]:
                if w not in seen and w not in vcs:
                    seen.add(w)
                    stack.append(w)
        return False

    for a in range(len(X)):
        for b in range(a + 1, len(X)):
            if not has_avoiding_path(X[a], X[b]):
                return True
    return False


def weight_sum(edges, wfine):
    """R29: sum over the distinct edges of round-half-up(w * 2^32), in exact rationals."""
    from fractions import Fraction
    tot = 0
    for e in set(int(x) for x in edges):
        q = Fraction(float(wfine[e])) * (1 << 32) + Fraction(1, 2)
        tot += q.numerator // q.denominator
    return tot


def search_plain(V, src, dst, act, central, marginal, k, depth, gamma=0.5, wfine=None):
    """Plain-definition form of the search (after R21):
    candidates = CGs identified by the central terminating level (ties kept, R13);
    marginal run exhaustive to depth D; attach all; PTC filter; sort (S^r, S^c, v); take k.
    With wfine (tie-break R29) the sort is (S^r, S^c, W(result edges), v)."""
    src = np.asarray(src)
    dst = np.asarray(dst)
    nc, nm = len(central), len(marginal)
    Hc = o2_levels(V, src, dst, act, central, depth, True)
    complete = (Hc != INF).all(axis=1)
    mx = np.where(complete, Hc.max(axis=1), INF)
    w = k
    Lend = depth
    for L in range(depth + 1):
        if (mx <= L).sum() >= w:
            Lend = L
            break
    cands = sorted((int(mx[v]), v) for v in range(V) if mx[v] <= Lend)
    bc = np.where(complete, mx, INF)
    # truncate H to the terminating level (values > Lend were never written)
    Hc_t = np.where(Hc <= Lend, Hc, INF)
    bc_t = np.where(bc <= Lend, bc, INF)
    cgs = []
    for sc, v in cands:
        ce, cn = set(), {v}
        for j in range(nc):
            e, n = enumerate_min_paths(V, src, dst, act, Hc_t, j, bc_t, [v])
            ce |= e
            cn |= n
        vcl = sorted(x for x in cn if (Hc_t[x] == 0).any())
        cgs.append((sc, v, ce, cn, vcl))
    res = []
    if nm == 0:
        for sc, v, ce, cn, vcl in cgs:
            res.append((float(sc), sc, v, 0, sorted(cn), sorted(ce), vcl, True))
    else:
        Hm = o2_levels(V, src, dst, act, marginal, depth, nm >= 2)
        cm = (Hm != INF).all(axis=1)
        bm = np.where(cm, Hm.max(axis=1), INF) if nm >= 2 else np.full(V, INF)
        for sc, v, ce, cn, vcl in cgs:
            D = [min(int(Hm[x, i]) for x in vcl) for i in range(nm)]
            if any(d == INF for d in D):
                continue
            sm = max(D)
            me, mn = set(), set()
            for i in range(nm):
                starts = [x for x in vcl if Hm[x, i] == D[i]]
                e, n = enumerate_min_paths(V, src, dst, act, Hm, i, bm, starts)
                me |= e
                mn |= n
            nodes = cn | mn
            edges = ce | me
            p = ptc_brute(V, src, dst, nodes, edges, vcl, Hm, nm)
            sr = gamma * float(sc) + (1.0 - gamma) * float(sm)
            res.append((sr, sc, v, sm, sorted(nodes), sorted(edges), vcl, p))
    res = [r for r in res if r[7]]
    if wfine is None:
        res.sort(key=lambda r: (r[0], r[1], r[2]))
    else:
        res.sort(key=lambda r: (r[0], r[1], weight_sum(r[5], wfine), r[2]))
    return res[:k], cands
