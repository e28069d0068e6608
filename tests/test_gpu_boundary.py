"""GPU checks of the C-ABI conventions (include/riki.h): the coarsening's ln matches the
oracle's libm log over the whole integer domain of label counts, one graph handle serves
concurrent callers, and a search runs on the caller's CUDA stream."""
import ctypes as C
import os
import subprocess
import threading

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def P():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_2001_06770_b200 as pkg
    return pkg


def _host_ln(tmp):
    so = os.path.join(tmp, "libln.so")
    subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC", "-shared",
                           os.path.join(ROOT, "tests", "c", "ln_table.c"), "-o", so, "-lquadmath", "-lm"])
    lib = C.CDLL(so)
    lib.host_ln_table.argtypes = [C.c_uint64, C.c_uint64, C.c_void_p]
    lib.host_ln_table.restype = None
    return lib


def test_coarsening_ln_correctly_rounded_exhaustively(P, tmp_path):
    # P:193 takes ln of the integer cA + cB; R31 fixes its fp64 value as the correctly rounded
    # one.  Both counts are at most the node's degree, so the domain is [2, 2 * max degree];
    # [1, 2^27) covers every graph with max degree < 2^26 (67M; config 4/5's largest hub has
    # ~2M).  The device's double-double ln must equal binary128 logq rounded once, bit for bit
    # (CUDA's own log() differs on ~1e-5 of these integers, glibc's log on ~3e-5).
    lib = _host_ln(str(tmp_path))
    chunk = 1 << 24
    host = np.empty(chunk, np.float64)
    for n0 in range(1, 1 << 27, chunk):
        cnt = min(chunk, (1 << 27) - n0)
        dev = P.riki.debug_ln_table(n0, cnt)
        lib.host_ln_table(n0, cnt, host.ctypes.data)
        d = np.nonzero(dev.view(np.uint64) != host[:cnt].view(np.uint64))[0]
        assert len(d) == 0, f"ln differs at n = {(n0 + d[:5]).tolist()}"
    # where glibc's log is not correctly rounded the device still is (exact decimal reference)
    from decimal import Decimal, getcontext
    getcontext().prec = 60
    for n in (9170, 136837, 141614, 147674, 277862, 330034, 351497):
        assert P.riki.debug_ln_table(n, 1)[0] == float(Decimal(n).ln())


def _c1_graph(P):
    kg = synth.make_kg(1)
    g = P.Graph(kg.n_nodes, kg.src, kg.dst, kg.label_class, kg.term_ptr, kg.postings)
    g.set_label_weights(0.5, kg.avg_hops)
    return kg, g


def _key(r):
    return [(x.central_node, x.sc, x.sm, x.score, x.nodes.tolist(), x.edge_ids.tolist()) for x in r.rpgs]


def test_concurrent_batches_on_one_handle_equal_serial(P):
    # Threading convention: one handle serves concurrent callers (ctypes releases the GIL, so
    # the calls really overlap on the host; the handle lock serialises them on the device)
    kg, g = _c1_graph(P)
    qs = synth.config_queries(kg, 1)
    halves = [(qs.central[:50], qs.marginal[:50]), (qs.central[50:], qs.marginal[50:])]
    serial = [g.search_batch(c, m, qs.k, qs.depth) for c, m in halves]
    for rounds in range(3):
        out = [None, None]
        errs = []

        def run(i):
            try:
                res = []
                for _ in range(4):
                    res = g.search_batch(halves[i][0], halves[i][1], qs.k, qs.depth)
                    g.search(halves[i][0][0], halves[i][1][0], qs.k, qs.depth)
                out[i] = res
            except Exception as e:  # pragma: no cover - reported below
                errs.append(e)

        th = [threading.Thread(target=run, args=(i,)) for i in range(2)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        assert not errs, errs
        for i in range(2):
            assert [_key(r) for r in out[i]] == [_key(r) for r in serial[i]]


def test_search_on_caller_stream(P):
    import torch
    kg, g = _c1_graph(P)
    qs = synth.config_queries(kg, 1, 12)
    s = torch.cuda.Stream()
    for i in range(12):
        a = g.search(qs.central[i], qs.marginal[i], qs.k, qs.depth)
        b = g.search(qs.central[i], qs.marginal[i], qs.k, qs.depth, stream=s.cuda_stream)
        assert _key(a) == _key(b)


def test_fetch_guard(P):
    # a device batch can be fetched once; any other call on the handle in between invalidates it
    import torch
    kg, g = _c1_graph(P)
    qs = synth.config_queries(kg, 1, 8)
    cp, ct = P.Graph._csr(qs.central)
    mp, mt = P.Graph._csr(qs.marginal)
    d = [torch.from_numpy(x.astype(np.int64 if x.dtype == np.uint64 else np.int32)).cuda() for x in (cp, ct, mp, mt)]
    n = len(qs.central)
    ncs, nms = [len(c) for c in qs.central], [len(m) for m in qs.marginal]
    g.search_batch_device(n, *(x.data_ptr() for x in d), qs.k, qs.depth)
    first = g.fetch(n, ncs, nms)
    with pytest.raises(P.RikiError):
        g.fetch(n, ncs, nms)
    g.search_batch_device(n, *(x.data_ptr() for x in d), qs.k, qs.depth)
    g.search(qs.central[0], qs.marginal[0], qs.k, qs.depth)
    with pytest.raises(P.RikiError):
        g.fetch(n, ncs, nms)
    assert len(first) == n
