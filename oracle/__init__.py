"""CPU oracle for RIKI (arXiv 2001.06770) -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_2001_06770_b200`` + ``libriki.so``) never imports it, and the two share
no code: the oracle is ``oracle/riki_oracle.c`` (plain single-threaded C, fp64,
``-ffp-contract=off``) driven through ctypes here.

Citations: P:n = PAPER.md line n.  Functions:
  fine_weights   P:193-194      coarsen     P:202-217 (Eq. 1-3)
  bound          P:242-251      path_score
  phase          P:341-464      search
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "riki_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

INF = 0xFF


def build(force: bool = False) -> str:
    """Compile the oracle (gcc -O2 -ffp-contract=off).  Building the checker is not using it."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                               "-shared", "-o", tmp, _SRC, "-lquadmath", "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is not None:
        return _lib
    lib = C.CDLL(build())
    P, u32, u64, i32, dbl = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int, C.c_double
    sig = {
        "orc_fine_weights": (i32, [u32, u64, P, P, P, P]),
        "orc_coarsen": (i32, [dbl, dbl, dbl]),
        "orc_ln_count": (dbl, [u64]),
        "orc_coarsen_all": (None, [u64, P, dbl, dbl, P]),
        "orc_bound": (None, [i32, dbl, dbl, P, P]),
        "orc_path_score": (i32, [P, i32]),
        "orc_rpg_score": (dbl, [dbl, u32, u32]),
        "orc_graph_new": (P, [u32, u64, P, P, P]),
        "orc_graph_free": (None, [P]),
        "orc_phase": (i32, [P, u32, P, P, u32, i32, P, P, P]),
        "orc_search": (P, [P, u32, P, P, u32, P, P, u32, u32, P]),
        "orc_result_free": (None, [P]),
        "orc_res_count": (u32, [P]),
        "orc_res_ncand": (u32, [P]),
        "orc_res_levels": (None, [P, P, P, P, P, P, P]),
        "orc_res_times": (None, [P, P, P]),
        "orc_res_cand": (None, [P, u32, P, P, P, P, P, P, P, P, P]),
        "orc_res_cand_lists": (None, [P, u32, P, P, P]),
        "orc_res_get": (None, [P, u32, P, P, P, P, P, P, P, P, P]),
        "orc_res_wsum": (C.c_uint64, [P, u32]),
        "orc_res_lists": (None, [P, u32, P, P, P, P, P]),
        "orc_res_matrix": (i32, [P, i32, P, P]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p) if a is not None and a.size else None


class _Params(C.Structure):
    _fields_ = [("gamma", C.c_double), ("beam_w", C.c_uint32), ("beam_mode", C.c_int),
                ("ptc_mode", C.c_int), ("early_term", C.c_int), ("tie_break", C.c_int), ("wfine", C.c_void_p)]


# ---------------------------------------------------------------- weighting
def fine_weights(n_nodes: int, src, dst, cls) -> np.ndarray:
    """w = ln(#same-class out-edges of src + #same-class in-edges of dst), min-max to [0,1]."""
    lib = _load()
    src = np.ascontiguousarray(src, np.uint32)
    dst = np.ascontiguousarray(dst, np.uint32)
    cls = np.ascontiguousarray(cls, np.uint32)
    out = np.zeros(len(src), np.float64)
    rc = lib.orc_fine_weights(n_nodes, len(src), _ptr(src), _ptr(dst), _ptr(cls), _ptr(out))
    if rc:
        raise MemoryError("oracle fine_weights")
    return out


def ln_count(n: int) -> float:
    """R31: ln of an integer count, correctly rounded to fp64 (P:193's log)."""
    return _load().orc_ln_count(n)


def coarsen(w: float, alpha: float, avg_hops: float) -> int:
    """Eq. 1-3 for one weight."""
    return _load().orc_coarsen(float(w), float(alpha), float(avg_hops))


def coarsen_all(w, alpha: float, avg_hops: float) -> np.ndarray:
    w = np.ascontiguousarray(w, np.float64)
    out = np.zeros(len(w), np.uint8)
    _load().orc_coarsen_all(len(w), _ptr(w), float(alpha), float(avg_hops), _ptr(out))
    return out


def bound(a: int, alpha: float, avg_hops: float):
    """Theorem boundEdgeWeight: [lo, hi) containing w given a."""
    lo, hi = C.c_double(), C.c_double()
    _load().orc_bound(int(a), float(alpha), float(avg_hops), C.byref(lo), C.byref(hi))
    return lo.value, hi.value


def path_score(seq) -> int:
    """Def. pathScoring."""
    a = np.ascontiguousarray(seq, np.int32)
    return _load().orc_path_score(_ptr(a), len(a))


def rpg_score(gamma: float, sc: int, sm: int) -> float:
    """Eq. 6."""
    return _load().orc_rpg_score(gamma, sc, sm)


# ---------------------------------------------------------------- graph / search
class Graph:
    """Oracle-side copy of a bidirected graph with activation levels a_e."""

    def __init__(self, n_nodes: int, src, dst, act):
        self.lib = _load()
        self.V = int(n_nodes)
        self.src = np.ascontiguousarray(src, np.uint32)
        self.dst = np.ascontiguousarray(dst, np.uint32)
        self.act = np.ascontiguousarray(act, np.uint8)
        self.E = len(self.src)
        self.h = self.lib.orc_graph_new(self.V, self.E, _ptr(self.src), _ptr(self.dst), _ptr(self.act))

    def __del__(self):
        if getattr(self, "h", None):
            self.lib.orc_graph_free(self.h)
            self.h = None


def _postings_csr(terms_nodes):
    ptr = np.zeros(len(terms_nodes) + 1, np.uint64)
    for i, t in enumerate(terms_nodes):
        ptr[i + 1] = ptr[i] + len(t)
    flat = np.concatenate([np.asarray(t, np.uint32) for t in terms_nodes]) if terms_nodes else np.zeros(0, np.uint32)
    return ptr, np.ascontiguousarray(flat, np.uint32)


def phase(g: Graph, terms_nodes, depth: int, block_mode: int):
    """Raw exploration (no termination besides depth / empty frontier).  block_mode:
    0 none, 1 central (CF when the row completes), 2 marginal stop rule (T>=2).
    Returns (H[V,T] uint8, block[V] uint8, L_end, relaxations)."""
    T = len(terms_nodes)
    ptr, flat = _postings_csr(terms_nodes)
    H = np.zeros((g.V, T), np.uint8)
    blk = np.zeros(g.V, np.uint8)
    rel = C.c_uint64()
    L = g.lib.orc_phase(g.h, T, _ptr(ptr), _ptr(flat), depth, block_mode, _ptr(H), _ptr(blk), C.byref(rel))
    return H, blk, int(L), int(rel.value)


@dataclass
class RPG:
    central_node: int
    sc: int
    sm: int
    score: float
    ptc: int
    nodes: np.ndarray
    edge_ids: np.ndarray
    vc: np.ndarray
    cdist: np.ndarray
    mdist: np.ndarray
    wsum: int = 0  # tie_break 1: W(G^r) in units of 2^-32 (R29)


@dataclass
class Candidate:
    v: int
    sc: int
    attached: int
    ptc: int
    sm: int
    sr: float
    cg_nodes: np.ndarray
    cg_edges: np.ndarray
    vc: np.ndarray


@dataclass
class SearchResult:
    rpgs: list
    candidates: list
    Lc: int
    Lm: int
    relax_c: int
    relax_m: int
    n_attached: int
    n_ptc_fail: int
    Hc: np.ndarray = None
    bc: np.ndarray = None
    Hm: np.ndarray = None
    bm: np.ndarray = None
    extra: dict = field(default_factory=dict)


def search(g: Graph, central_nodes, marginal_nodes, k: int, depth: int, gamma: float = 0.5, beam_w: int = 0,
           beam_mode: int = 0, ptc_mode: int = 0, early_term: int = 0, want_matrices: bool = True,
           want_candidates: bool = True, tie_break: int = 0, wfine=None) -> SearchResult:
    """Full RPQ search (Def. RPKSP).  central_nodes / marginal_nodes are
    lists of posting lists (one per keyword).  tie_break 1 (R29) ranks equal
    (S^r, S^c) by the weight sum of the result's distinct edges; wfine = the fine edge
    weights (f64 by edge id) it needs."""
    if not central_nodes:
        raise ValueError("C must be non-empty (Def. RPQ, P:105)")
    if k < 1:
        raise ValueError("k >= 1")
    lib = g.lib
    cp, cf = _postings_csr(central_nodes)
    mp, mf = _postings_csr(marginal_nodes)
    wf = None
    if tie_break:
        if wfine is None:
            raise ValueError("tie_break 1 needs the fine edge weights")
        wf = np.ascontiguousarray(wfine, np.float64)
        assert len(wf) == g.E
    prm = _Params(gamma, beam_w, beam_mode, ptc_mode, early_term, tie_break, wf.ctypes.data if wf is not None else None)
    r = lib.orc_search(g.h, len(central_nodes), _ptr(cp), _ptr(cf), len(marginal_nodes), _ptr(mp), _ptr(mf),
                       k, depth, C.byref(prm))
    try:
        nc, nm = len(central_nodes), len(marginal_nodes)
        Lc, Lm = C.c_int(), C.c_int()
        rc, rm = C.c_uint64(), C.c_uint64()
        na, nf = C.c_uint32(), C.c_uint32()
        lib.orc_res_levels(r, C.byref(Lc), C.byref(Lm), C.byref(rc), C.byref(rm), C.byref(na), C.byref(nf))
        out = SearchResult([], [], Lc.value, Lm.value, rc.value, rm.value, na.value, nf.value)
        tc, tm = C.c_double(), C.c_double()
        lib.orc_res_times(r, C.byref(tc), C.byref(tm))
        out.extra["t_central"], out.extra["t_marginal"] = tc.value, tm.value
        u32, u64, i32, dbl = C.c_uint32, C.c_uint64, C.c_int, C.c_double
        for i in range(lib.orc_res_count(r)):
            ci, v, sc, sm, sr, ptc = u32(), u32(), u32(), u32(), dbl(), i32()
            nn, ne, nv = u64(), u64(), u64()
            lib.orc_res_get(r, i, *(C.byref(x) for x in (ci, v, sc, sm, sr, ptc, nn, ne, nv)))
            nodes = np.zeros(nn.value, np.uint32)
            edges = np.zeros(ne.value, np.uint64)
            vc = np.zeros(nv.value, np.uint32)
            cd = np.zeros(nc, np.uint8)
            md = np.zeros(nm, np.uint8)
            lib.orc_res_lists(r, i, _ptr(nodes), _ptr(edges), _ptr(vc), _ptr(cd), _ptr(md))
            out.rpgs.append(RPG(v.value, sc.value, sm.value, sr.value, ptc.value, nodes, edges, vc, cd, md,
                                int(lib.orc_res_wsum(r, i))))
        if want_candidates:
            for i in range(lib.orc_res_ncand(r)):
                v, sc, sm = u32(), u32(), u32()
                att, ptc = i32(), i32()
                sr = dbl()
                ncn, nce, nvc = u64(), u64(), u64()
                lib.orc_res_cand(r, i, *(C.byref(x) for x in (v, sc, att, ptc, sm, sr, ncn, nce, nvc)))
                cn = np.zeros(ncn.value, np.uint32)
                ce = np.zeros(nce.value, np.uint64)
                vc = np.zeros(nvc.value, np.uint32)
                lib.orc_res_cand_lists(r, i, _ptr(cn), _ptr(ce), _ptr(vc))
                out.candidates.append(Candidate(v.value, sc.value, att.value, ptc.value, sm.value, sr.value,
                                                cn, ce, vc))
        if want_matrices:
            out.Hc = np.zeros((g.V, nc), np.uint8)
            out.bc = np.zeros(g.V, np.uint8)
            lib.orc_res_matrix(r, 0, _ptr(out.Hc), _ptr(out.bc))
            if nm:
                out.Hm = np.zeros((g.V, nm), np.uint8)
                out.bm = np.zeros(g.V, np.uint8)
                lib.orc_res_matrix(r, 1, _ptr(out.Hm), _ptr(out.bm))
        return out
    finally:
        lib.orc_result_free(r)


# ---------------------------------------------------------------- Abar by sampled pairs
HOP_INF = 0xFFFFFFFF


def sample_avg_hops(n_nodes: int, src, dst, ps, pt, max_hops: int = 255):
    """P:611 "We sample ten thousand pairs of nodes for estimation of Abar" (Abar: "the average
    shortest hops in the graph").  Reading R30: d(s, t) = fewest edges of a directed path
    s -> t in the edge list (BFS; scipy's unweighted shortest_path is the BFS step), pairs with no
    path within max_hops are left out; mean and sample standard deviation (n - 1) from exact
    integer moments: mean = S1 / n, sd = sqrt((n*S2 - S1^2) / (n * (n - 1))).
    Returns (mean, sd, n_reached, dist[] with HOP_INF for no path)."""
    import math

    import scipy.sparse as sp
    import scipy.sparse.csgraph as cg
    src = np.asarray(src, np.int64)
    dst = np.asarray(dst, np.int64)
    ps = np.asarray(ps, np.int64)
    pt = np.asarray(pt, np.int64)
    dist = np.full(len(ps), HOP_INF, np.uint32)
    if len(ps):
        A = sp.csr_matrix((np.ones(len(src)), (src, dst)), shape=(n_nodes, n_nodes))
        uniq = np.unique(ps)
        row = {int(x): i for i, x in enumerate(uniq)}
        D = cg.shortest_path(A, directed=True, unweighted=True, indices=uniq)
        for i, (s_, t_) in enumerate(zip(ps, pt)):
            d = D[row[int(s_)], int(t_)]
            if np.isfinite(d) and d <= max_hops:
                dist[i] = int(d)
    ok = [int(x) for x in dist if x != HOP_INF]
    n = len(ok)
    s1 = sum(ok)
    s2 = sum(x * x for x in ok)
    mean = float(s1) / float(n) if n else float("nan")
    sd = math.sqrt(float(n * s2 - s1 * s1) / (float(n) * float(n - 1))) if n >= 2 else float("nan")
    return mean, sd, n, dist
