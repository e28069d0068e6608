"""Vertex-partitioned mode (include/riki.h riki_dist_*).

CPU (`-m "not gpu"`): the partition bounds (host-only riki_dist_partition) against a brute-force
restatement of their definition; the rank-0 unique-id broadcast of dist.init_vertex_partitioned
over a world-size-2 gloo group.

GPU (`-m gpu`): the partitioned path must give the oracle's H / block / relaxation counts and
the oracle's search results bit for bit -- with nranks partitions simulated in one process
(every partition's push -- its owned frontier nodes' out-edges OR-ed into the owners' bit-plane
slices, the fused exchange -- runs on the one GPU; the exchange is the identity), and through
a real 1-rank NCCL communicator.  The earlier pull variant (RIKI_VP_PULL=1: every rank pulls
its owned range, one all-gather per level) is checked the same way."""
import os
import socket

import numpy as np
import pytest

import oracle as O
import synth
from fixtures import random_instance

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ------------------------------------------------------------------------------ CPU: bounds
def _brute_bounds(irow, P):
    """bounds[r] = the smallest multiple of 32 (capped at V) whose prefix weight
    sum_{v < b} (indeg(v) + 1) reaches ceil(total * r / P)."""
    V = len(irow) - 1
    w = np.diff(irow.astype(np.int64)) + 1
    pre = np.concatenate([[0], np.cumsum(w)])
    total = int(pre[-1])
    out = [0]
    for r in range(1, P):
        target = -(-total * r // P)
        b = 0
        while b < V and pre[b] < target:
            b += 1
        out.append(min(-(-b // 32) * 32, V))
    out.append(V)
    return np.array(out, np.uint32)


@pytest.mark.parametrize("seed", range(12))
def test_partition_bounds_match_definition(seed):
    import paper_2001_06770_b200.riki as R
    rng = np.random.default_rng(900 + seed)
    V = int(rng.choice([0, 1, 31, 32, 33, 100, 1000, 4096]))
    deg = (rng.pareto(1.2, V) * 3).astype(np.int64)
    irow = np.concatenate([[0], np.cumsum(deg)]).astype(np.uint32)
    for P in (1, 2, 3, 5, 8, 64):
        b = R.dist_partition(irow, P)
        assert b.tolist() == _brute_bounds(irow, P).tolist()
        assert b[0] == 0 and b[-1] == V and (np.diff(b.astype(np.int64)) >= 0).all()
        assert all(x % 32 == 0 or x == V for x in b)
        # balance: a range exceeds its share by at most the 32-node alignment window
        w = np.diff(irow.astype(np.int64)) + 1
        pre = np.concatenate([[0], np.cumsum(w)])
        win = max((pre[min(i + 32, V)] - pre[i] for i in range(0, V + 1, 32)), default=0)
        for r in range(P):
            assert pre[b[r + 1]] - pre[b[r]] <= -(-int(pre[-1]) // P) + win + 1


def test_partition_rejects_bad_input():
    import paper_2001_06770_b200.riki as R
    with pytest.raises(R.RikiError):
        R.dist_partition(np.array([0, 5, 3], np.uint32), 2)
    with pytest.raises(R.RikiError):
        R.dist_partition(np.array([0, 1], np.uint32), 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class _FakeGraph:
    def __init__(self):
        self.calls = []

    def dist_init(self, nranks, rank, uid, mode=1):
        self.calls.append((nranks, rank, uid, mode))


def _vp_worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2001_06770_b200 import dist as D
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = _FakeGraph()
    uid = bytes(range(128))
    D.init_vertex_partitioned(g, unique_id_fn=(lambda: uid) if rank == 0 else (lambda: b"x" * 128))
    q.put((rank, g.calls))
    dist.destroy_process_group()


def test_init_vertex_partitioned_gloo_world2():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_vp_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    uid = bytes(range(128))
    assert got[0] == [(2, 0, uid, 1)] and got[1] == [(2, 1, uid, 1)]


# ------------------------------------------------------------------------------ GPU parity
@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2001_06770_b200 as pkg
    return pkg


def _dev_graph(P, V, src, dst, act, postings):
    tp = np.zeros(len(postings) + 1, np.uint64)
    tp[1:] = np.cumsum([len(x) for x in postings])
    po = np.concatenate([np.asarray(x, np.uint32) for x in postings])
    g = P.Graph(V, src, dst, None, tp, po)
    g.set_activation_levels(act)
    return g


def _cmp(a_res, b_res):
    assert len(a_res.rpgs) == len(b_res.rpgs)
    for a, b in zip(a_res.rpgs, b_res.rpgs):
        assert (a.central_node, a.sc, a.sm, a.ptc, a.score) == (b.central_node, b.sc, b.sm, b.ptc, b.score)
        assert a.nodes.tolist() == b.nodes.tolist() and a.edge_ids.tolist() == b.edge_ids.tolist()
        assert a.vc.tolist() == b.vc.tolist()


def _hub_graph(rng, V=3000, m=9000):
    hubs = rng.integers(0, V, 12)
    u = rng.integers(0, V, m)
    v = np.where(rng.random(m) < 0.4, hubs[rng.integers(0, 12, m)], rng.integers(0, V, m))
    v = np.where(u == v, (v + 1) % V, v)
    src = np.empty(2 * m, np.uint32)
    dst = np.empty(2 * m, np.uint32)
    src[0::2], dst[0::2] = u, v
    src[1::2], dst[1::2] = v, u
    act = rng.integers(0, 5, 2 * m).astype(np.uint8)
    return V, src, dst, act


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("nranks", [2, 3, 8])
@pytest.mark.parametrize("variant", ["push", "pull"])
def test_vp_simulated_hitting_levels(P, seed, nranks, variant, monkeypatch):
    if variant == "pull":
        monkeypatch.setenv("RIKI_VP_PULL", "1")  # read by riki_dist_init
    rng = np.random.default_rng(9100 + seed)
    if seed % 2:
        V, src, dst, act = _hub_graph(rng)
        post = [np.unique(rng.integers(0, V, int(rng.integers(1, 30)))).astype(np.uint32) for _ in range(8)]
    else:
        V, src, dst, act, post = random_instance(rng, 40, 400, deg=3.0, T_hi=8, post_hi=6)
    g = _dev_graph(P, V, src, dst, act, post)
    g.dist_init(nranks, 0, None, mode=1)
    info = g.dist_info()
    assert info["mode"] == 1 and info["nranks"] == nranks and info["bounds"][-1] == V
    og = O.Graph(V, src, dst, act)
    T = min(len(post), 8)
    for D in (3, 20):
        for mode in (0, 1, 2):
            H, blk, rel, L = g.hitting_levels(np.arange(T, dtype=np.uint32), D, mode)
            Ho, bo, Lo, relo = O.phase(og, post[:T], D, mode)
            assert (H == Ho).all(), (D, mode, np.argwhere(H != Ho)[:5])
            assert (blk == bo).all() and L == Lo and rel == relo
    assert g.dist_info()["exchanges"] > 0


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(10))
def test_vp_simulated_search_random(P, seed):
    rng = np.random.default_rng(9300 + seed)
    V, src, dst, act, _ = random_instance(rng, 30, 200, deg=3.0, amax=4)
    nterm = 10
    post = [np.unique(rng.integers(0, V, int(rng.integers(1, 4)))).astype(np.uint32) for _ in range(nterm)]
    g = _dev_graph(P, V, src, dst, act, post)
    g.dist_init(int(rng.choice([2, 4, 7])), 0, None, mode=1)
    og = O.Graph(V, src, dst, act)
    for _ in range(4):
        nc = int(rng.integers(1, 4))
        nm = int(rng.integers(0, 4))
        tt = rng.choice(nterm, nc + nm, replace=False)
        C, M = tt[:nc], tt[nc:]
        k = int(rng.choice([1, 3, 5]))
        D = int(rng.choice([3, 6, 20]))
        kw = dict(ptc_mode=int(rng.integers(0, 4)), early_term=int(rng.integers(0, 3)))
        r = g.search(C, M, k, D, **kw)
        ro = O.search(og, [post[t] for t in C], [post[t] for t in M], k, D, **kw)
        assert len(r.rpgs) == len(ro.rpgs)
        for a, b in zip(r.rpgs, ro.rpgs):
            assert (a.central_node, a.sc, a.sm, a.ptc, a.score) == (b.central_node, b.sc, b.sm, b.ptc, b.score)
            assert a.nodes.tolist() == b.nodes.tolist() and a.edge_ids.tolist() == b.edge_ids.tolist()
        assert r.stats["relax_central"] == ro.relax_c and r.stats["relax_marginal"] == ro.relax_m


@pytest.mark.gpu
def test_vp_c1_batch_simulated_and_nccl_one_rank(P):
    kg = synth.make_kg(1)
    qs = synth.config_queries(kg, 1)
    g = P.Graph(kg.n_nodes, kg.src, kg.dst, kg.label_class, kg.term_ptr, kg.postings)
    g.set_label_weights(0.5, kg.avg_hops)
    og = O.Graph(kg.n_nodes, kg.src, kg.dst, O.coarsen_all(O.fine_weights(kg.n_nodes, kg.src, kg.dst, kg.label_class), 0.5, kg.avg_hops))
    base = g.search_batch(qs.central, qs.marginal, qs.k, qs.depth)
    for i in range(0, len(base), 9):
        ro = O.search(og, [kg.posting(t) for t in qs.central[i]], [kg.posting(t) for t in qs.marginal[i]], qs.k,
                      qs.depth)
        _cmp(base[i], ro)
    g.dist_init(5, 0, None, mode=1)  # simulated: 5 partitions on this GPU
    for a, b in zip(g.search_batch(qs.central, qs.marginal, qs.k, qs.depth), base):
        _cmp(a, b)
    import torch  # noqa: F401  (loads torch's NCCL, which riki_dist_* then shares)
    g.dist_init(1, 0, P.riki.dist_unique_id(), mode=1)  # real NCCL communicator, 1 rank
    assert g.dist_info()["nranks"] == 1
    for a, b in zip(g.search_batch(qs.central, qs.marginal, qs.k, qs.depth), base):
        _cmp(a, b)
    assert g.dist_info()["exchanges"] > 0
    with pytest.raises(P.RikiError):
        g.set_joint(True)
    g.dist_init(1, 0, None, mode=0)  # back to replicated
    for a, b in zip(g.search_batch(qs.central, qs.marginal, qs.k, qs.depth), base):
        _cmp(a, b)


@pytest.mark.gpu
@pytest.mark.slow
def test_vp_c2_sampled_queries(P):
    # config 2 at full size (1M nodes / 5M edges), 8 simulated partitions: the partitioned path
    # gives the replicated path's results; 2 queries also against the oracle
    kg = synth.make_kg(2)
    qs = synth.config_queries(kg, 2, 24)
    g = P.Graph(kg.n_nodes, kg.src, kg.dst, kg.label_class, kg.term_ptr, kg.postings)
    g.set_label_weights(0.5, kg.avg_hops)
    base = g.search_batch(qs.central, qs.marginal, qs.k, qs.depth)
    g.dist_init(8, 0, None, mode=1)
    vp = g.search_batch(qs.central, qs.marginal, qs.k, qs.depth)
    for a, b in zip(vp, base):
        _cmp(a, b)
        assert a.stats["relax_central"] == b.stats["relax_central"]
        assert a.stats["relax_marginal"] == b.stats["relax_marginal"]
    og = O.Graph(kg.n_nodes, kg.src, kg.dst, O.coarsen_all(O.fine_weights(kg.n_nodes, kg.src, kg.dst, kg.label_class), 0.5, kg.avg_hops))
    for i in (0, 13):
        ro = O.search(og, [kg.posting(t) for t in qs.central[i]], [kg.posting(t) for t in qs.marginal[i]], qs.k,
                      qs.depth, want_matrices=False)
        _cmp(vp[i], ro)
