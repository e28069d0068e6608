"""Seeded synthetic knowledge graphs and RPQ query sets (input recipe).

This module is the ONLY code shared by the oracle side and the CUDA side, and
it holds none of the method's arithmetic: no weights, no coarsening, no search.
It produces

* a bidirected labelled multigraph as a directed edge list (src, dst,
  label_class) with one reverse edge per triple (class = 2*label +
  inverse flag),
* a keyword -> node inverted index (term_ptr, postings; sorted, unique),
* query sets (central term ids, marginal term ids),

with the shapes of the paper's workloads (Table 1, Table 3
P:706-732, Table 2) scaled to BASELINE.json's configs.
Graph seed = 1000 + config number, query seed = 2000 + config number.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class KG:
    n_nodes: int
    src: np.ndarray        # uint32 [E] directed, reverse edges included
    dst: np.ndarray        # uint32 [E]
    label_class: np.ndarray  # uint32 [E] = 2*label + inverse flag
    term_ptr: np.ndarray   # uint64 [n_terms+1]
    postings: np.ndarray   # uint32 [sum |V_t|], each term's list sorted unique
    avg_hops: float        # A-bar used by the coarsening (an input parameter, R4)
    n_labels: int

    @property
    def n_edges(self) -> int:
        return int(len(self.src))

    @property
    def n_terms(self) -> int:
        return int(len(self.term_ptr) - 1)

    def posting(self, t: int) -> np.ndarray:
        return self.postings[int(self.term_ptr[t]):int(self.term_ptr[t + 1])]


@dataclass
class QuerySet:
    central: list   # list of lists of term ids
    marginal: list  # list of lists of term ids
    k: int
    depth: int


@dataclass
class ConfigSpec:
    name: str
    n_nodes: int
    n_edges: int          # directed CSR entries after adding reverse edges (R26)
    n_labels: int
    n_central: int
    n_marginal: int
    k: int
    depth: int
    n_queries: int
    post_lo: int
    post_hi: int
    n_terms: int
    avg_hops: float | None  # None -> exact all-pairs mean (tiny config only)
    degree_postings: bool = False


# BASELINE.json configs (index = config number - 1); SURVEY §8.0 / §8(d)
def _scaled(lo, hi, V, Vp):
    return max(1, int(round(lo * V / Vp))), max(2, int(round(hi * V / Vp)))


CONFIGS = {
    1: ConfigSpec("tiny", 200, 800, 8, 2, 1, 3, 3, 100, 1, 5, 48, None),
    2: ConfigSpec("powerlaw-1M", 1_000_000, 5_000_000, 200, 2, 2, 10, 20, 200,
                  *_scaled(5, 6059, 1_000_000, 15.1e6), 4096, 3.87),
    3: ConfigSpec("dbpedia-5M", 5_000_000, 20_000_000, 1000, 3, 3, 20, 20, 1000,
                  *_scaled(5, 6059, 5_000_000, 15.1e6), 8192, 3.87),
    4: ConfigSpec("wikidata-30M", 30_000_000, 150_000_000, 2000, 2, 4, 20, 20, 200,
                  *_scaled(51, 87102, 30_000_000, 30.6e6), 1024, 3.68, True),
    # C5: config 4's graph (same seed) with a 10k-query throughput batch: half 2 + 4, half the
    # Exp-1 mix cknum x mknum in {1,2,4} x {2,4,6} -- see c5_queries
    5: ConfigSpec("wikidata-30M-throughput", 30_000_000, 150_000_000, 2000, 2, 4, 20, 20, 10_000,
                  *_scaled(51, 87102, 30_000_000, 30.6e6), 1024, 3.68, True),
}
GRAPH_OF = {5: 4}  # configs that share another config's graph (and its seed)


def _chung_lu_weights(rng, n, exponent):
    # expected degree ~ i^(-1/(exponent-1)); ids randomly permuted afterwards
    i = np.arange(n, dtype=np.float64)
    w = (i + 1.0) ** (-1.0 / (exponent - 1.0))
    return w / w.sum()


def _searchsorted_right(cdf, x):
    """np.searchsorted(cdf, x, side="right"), identical result; torch's CPU kernel runs it on
    every host core (the 30M-node configs draw 75M endpoints per side)."""
    if len(x) >= 1 << 12:
        try:
            import torch
            return torch.searchsorted(torch.from_numpy(np.ascontiguousarray(cdf)),
                                      torch.from_numpy(np.ascontiguousarray(x)), right=True).numpy()
        except ImportError:
            pass
    return np.searchsorted(cdf, x, side="right")


def _sample(rng, p, size):
    # inverse-CDF sampling (equivalent in law to an alias table), deterministic per seed
    cdf = np.cumsum(p)
    cdf[-1] = 1.0
    return _searchsorted_right(cdf, rng.random(size)).astype(np.int64)


def make_graph(n_nodes: int, n_edges: int, n_labels: int, seed: int, *, in_exp: float = 2.1,
               out_exp: float = 2.5, zipf_s: float = 1.3, hub_frac: float = 1e-4, hub_p: float = 0.8):
    """Chung-Lu power-law directed multigraph with Zipf labels and label-correlated hubs.
    Returns (src, dst, label_class) with E = n_edges directed entries (n_edges/2 triples)."""
    assert n_edges % 2 == 0
    rng = np.random.default_rng(seed)
    m = n_edges // 2
    pin = _chung_lu_weights(rng, n_nodes, in_exp)
    pout = _chung_lu_weights(rng, n_nodes, out_exp)
    perm_in = rng.permutation(n_nodes)
    perm_out = rng.permutation(n_nodes)
    u = perm_out[_sample(rng, pout, m)]
    v = perm_in[_sample(rng, pin, m)]
    # drop self-loops by resampling (multi-edges kept)
    for _ in range(100):
        bad = np.nonzero(u == v)[0]
        if not len(bad):
            break
        u[bad] = perm_out[_sample(rng, pout, len(bad))]
        v[bad] = perm_in[_sample(rng, pin, len(bad))]
    bad = u == v
    v[bad] = (u[bad] + 1) % n_nodes
    # Zipf(s) labels
    lp = (np.arange(n_labels, dtype=np.float64) + 1.0) ** (-zipf_s)
    lp /= lp.sum()
    lab = _sample(rng, lp, m)
    # hubs (top hub_frac of in-weight) attract their own class label with prob hub_p
    n_hubs = max(1, int(n_nodes * hub_frac))
    hubs = perm_in[:n_hubs]
    hub_label = rng.integers(0, n_labels, n_hubs)
    hub_of = np.full(n_nodes, -1, np.int64)
    hub_of[hubs] = np.arange(n_hubs)
    hv = hub_of[v]
    sel = (hv >= 0) & (rng.random(m) < hub_p)
    lab[sel] = hub_label[hv[sel]]
    src = np.empty(2 * m, np.uint32)
    dst = np.empty(2 * m, np.uint32)
    cls = np.empty(2 * m, np.uint32)
    src[0::2], dst[0::2], cls[0::2] = u, v, 2 * lab          # original edge
    src[1::2], dst[1::2], cls[1::2] = v, u, 2 * lab + 1      # reverse edge
    return src, dst, cls


def make_postings(n_nodes: int, n_terms: int, lo: int, hi: int, seed: int, degree=None):
    """Inverted index with log-uniform posting sizes in [lo, hi] (Table 3 frequencies scaled);
    members uniform, or proportional to degree ("high-degree keyword nodes", config 4)."""
    rng = np.random.default_rng(seed)
    hi = min(hi, n_nodes)
    lo = min(lo, hi)
    sizes = np.exp(rng.uniform(np.log(lo), np.log(hi + 1), n_terms)).astype(np.int64)
    sizes = np.clip(sizes, lo, hi)
    cdf = None
    if degree is not None:
        cdf = np.cumsum(degree.astype(np.float64) + 1.0)
        cdf /= cdf[-1]
    ptr = np.zeros(n_terms + 1, np.uint64)
    lists = []
    for t in range(n_terms):
        s = int(sizes[t])
        nodes = np.zeros(0, np.int64)
        for _ in range(8):  # draw with replacement, keep unique, top up
            if cdf is None:
                draw = rng.integers(0, n_nodes, 2 * s + 8)
            else:
                draw = _searchsorted_right(cdf, rng.random(2 * s + 8))
            nodes = np.unique(np.concatenate([nodes, draw]))
            if len(nodes) >= s:
                break
        if len(nodes) > s:
            nodes = np.sort(rng.choice(nodes, size=s, replace=False))
        nodes = nodes.astype(np.uint32)
        lists.append(nodes)
        ptr[t + 1] = ptr[t] + len(nodes)
    return ptr, np.concatenate(lists).astype(np.uint32)


def exact_avg_hops(n_nodes, src, dst):
    """Mean undirected hop distance over connected ordered pairs (tiny config only).
    This is a workload PARAMETER (A-bar is an input, R4), computed by plain BFS."""
    from scipy.sparse import csr_matrix
    from scipy.sparse.csgraph import shortest_path
    A = csr_matrix((np.ones(len(src)), (src.astype(np.int64), dst.astype(np.int64))), shape=(n_nodes, n_nodes))
    d = shortest_path(A, unweighted=True, directed=False)
    mask = np.isfinite(d) & (d > 0)
    return float(d[mask].mean()) if mask.any() else 1.0


def make_kg(cfg: int | ConfigSpec, seed: int | None = None) -> KG:
    if isinstance(cfg, int):
        cfg = GRAPH_OF.get(cfg, cfg)
    spec = CONFIGS[cfg] if isinstance(cfg, int) else cfg
    num = cfg if isinstance(cfg, int) else 0
    seed = 1000 + num if seed is None else seed
    src, dst, cls = make_graph(spec.n_nodes, spec.n_edges, spec.n_labels, seed)
    deg = None
    if spec.degree_postings:
        deg = np.bincount(src, minlength=spec.n_nodes)
    tp, po = make_postings(spec.n_nodes, spec.n_terms, spec.post_lo, spec.post_hi, seed + 7, deg)
    avg = spec.avg_hops if spec.avg_hops is not None else exact_avg_hops(spec.n_nodes, src, dst)
    return KG(spec.n_nodes, src, dst, cls, tp, po, avg, spec.n_labels)


def make_queries(kg: KG, n_queries: int, n_central: int, n_marginal: int, k: int, depth: int,
                 seed: int) -> QuerySet:
    """Random distinct term ids per query (first terms central, rest marginal)."""
    rng = np.random.default_rng(seed)
    cs, ms = [], []
    for _ in range(n_queries):
        t = rng.choice(kg.n_terms, size=n_central + n_marginal, replace=False)
        cs.append([int(x) for x in t[:n_central]])
        ms.append([int(x) for x in t[n_central:]])
    return QuerySet(cs, ms, k, depth)


def c5_queries(kg: KG, n_queries: int, seed: int = 2005) -> QuerySet:
    """Config 5's batch: even queries 2 central + 4 marginal, odd queries drawn from the
    Exp-1 mix cknum in {1, 2, 4} x mknum in {2, 4, 6}; k = 20, D = 20."""
    rng = np.random.default_rng(seed)
    cs, ms = [], []
    for i in range(n_queries):
        nc, nm = (2, 4) if i % 2 == 0 else (int(rng.choice([1, 2, 4])), int(rng.choice([2, 4, 6])))
        t = rng.choice(kg.n_terms, size=nc + nm, replace=False)
        cs.append([int(x) for x in t[:nc]])
        ms.append([int(x) for x in t[nc:]])
    return QuerySet(cs, ms, 20, 20)


def config_queries(kg: KG, cfg: int, n_queries: int | None = None) -> QuerySet:
    if cfg == 5:
        return c5_queries(kg, n_queries or CONFIGS[5].n_queries)
    spec = CONFIGS[cfg]
    return make_queries(kg, n_queries or spec.n_queries, spec.n_central, spec.n_marginal, spec.k, spec.depth,
                        2000 + cfg)


def random_small_kg(seed: int, n_nodes: int, n_edges: int, n_labels: int = 4, n_terms: int = 8,
                    post_hi: int = 3) -> KG:
    """Tiny uniform random bidirected graph for parity/property tests."""
    rng = np.random.default_rng(seed)
    m = n_edges // 2
    u = rng.integers(0, n_nodes, m)
    v = rng.integers(0, n_nodes, m)
    v = np.where(u == v, (v + 1) % n_nodes, v)
    lab = rng.integers(0, n_labels, m)
    src = np.empty(2 * m, np.uint32); dst = np.empty(2 * m, np.uint32); cls = np.empty(2 * m, np.uint32)
    src[0::2], dst[0::2], cls[0::2] = u, v, 2 * lab
    src[1::2], dst[1::2], cls[1::2] = v, u, 2 * lab + 1
    tp, po = make_postings(n_nodes, n_terms, 1, post_hi, seed + 1)
    return KG(n_nodes, src, dst, cls, tp, po, 3.0, n_labels)
