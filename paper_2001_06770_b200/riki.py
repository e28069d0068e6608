"""Thin ctypes binding of libriki.so (include/riki.h).  Argument marshalling only: every
step of the search runs in the library's CUDA kernels.  If libriki.so is missing this
module raises -- there is no CPU fallback (build it with ``python -m
paper_2001_06770_b200.build`` or ``__graft_entry__.build()``)."""
from __future__ import annotations

import ctypes as C
import os
import re
from collections.abc import Sequence
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("RIKI_LIB", os.path.join(HERE, "libriki.so"))
HEADER = os.path.join(os.path.dirname(HERE), "include", "riki.h")

STATUS = {0: "RIKI_OK", -1: "RIKI_EINVAL", -2: "RIKI_ENOMEM", -3: "RIKI_ECUDA", -4: "RIKI_EEMPTY_CENTRAL",
          -5: "RIKI_EUNRESOLVED", -6: "RIKI_ENOWEIGHTS", -7: "RIKI_EDEPTH", -8: "RIKI_ENCCL", -9: "RIKI_ENOSYS"}

_lib = None


class RikiError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code
        self.name = STATUS.get(code, str(code))


class Params(C.Structure):
    _fields_ = [("gamma", C.c_double), ("beam_w", C.c_uint32), ("beam_mode", C.c_int), ("tie_break", C.c_int),
                ("ptc_mode", C.c_int), ("early_term", C.c_int)]


class RPGStruct(C.Structure):
    _fields_ = [("central_node", C.c_uint32), ("sc", C.c_uint32), ("sm", C.c_uint32), ("score", C.c_double),
                ("ptc", C.c_uint8), ("n_nodes", C.c_uint32), ("nodes", C.POINTER(C.c_uint32)),
                ("n_edges", C.c_uint32), ("edge_ids", C.POINTER(C.c_uint64)), ("n_vc", C.c_uint32),
                ("vc", C.POINTER(C.c_uint32)), ("cdist", C.POINTER(C.c_uint8)), ("mdist", C.POINTER(C.c_uint8))]


class QueryStats(C.Structure):
    _fields_ = [("L_central", C.c_int32), ("L_marginal", C.c_int32), ("n_candidates", C.c_uint32),
                ("n_attached", C.c_uint32), ("n_ptc_fail", C.c_uint32), ("relax_central", C.c_uint64),
                ("relax_marginal", C.c_uint64)]


# numpy view of QueryStats (same layout as the C struct, checked at import)
_STATS_DT = np.dtype([(f, np.dtype(t)) for f, t in (("L_central", np.int32), ("L_marginal", np.int32),
                                                    ("n_candidates", np.uint32), ("n_attached", np.uint32),
                                                    ("n_ptc_fail", np.uint32), ("relax_central", np.uint64),
                                                    ("relax_marginal", np.uint64))], align=True)
assert _STATS_DT.itemsize == C.sizeof(QueryStats) and all(
    _STATS_DT.fields[f][1] == getattr(QueryStats, f).offset for f, _ in QueryStats._fields_)


class ExportSizes(C.Structure):
    _fields_ = [("n_rpg", C.c_uint64), ("n_nodes", C.c_uint64), ("n_edges", C.c_uint64), ("n_vc", C.c_uint64)]


class Stats(C.Structure):
    _fields_ = [("expand_launches", C.c_uint64), ("expand_ms", C.c_double), ("expand_bytes", C.c_uint64),
                ("relaxations", C.c_uint64), ("kernel_launches", C.c_uint64), ("queries", C.c_uint64),
                ("section_ms", C.c_double * 4), ("levels", C.c_uint64), ("retries", C.c_uint64),
                ("reallocs", C.c_uint64), ("exp_items", C.c_uint64), ("exp_items_work", C.c_uint64),
                ("exp_edges", C.c_uint64), ("exp_new_cells", C.c_uint64), ("exp_enqueued", C.c_uint64),
                ("exp_atomics", C.c_uint64)]


def declared_symbols():
    """Function names declared in include/riki.h (for the export check)."""
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(riki_\w+)\s*\(", txt)))


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libriki.so not built at {LIB_PATH}; run `python -m paper_2001_06770_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    P, u32, u64, i32, dbl = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int, C.c_double
    sig = {
        "riki_load_graph": (i32, [i32, u32, u64, P, P, P, u32, P, P, P]),
        "riki_load_graph_device": (i32, [i32, u32, u64, P, P, P, u32, P, P, P]),
        "riki_free_graph": (None, [P]),
        "riki_set_edge_weights": (i32, [P, P, dbl, dbl]),
        "riki_set_node_weights": (i32, [P, P, dbl, dbl]),
        "riki_set_label_weights": (i32, [P, dbl, dbl]),
        "riki_set_activation_levels": (i32, [P, P]),
        "riki_get_activation_levels": (i32, [P, P]),
        "riki_params_default": (None, [P]),
        "riki_rpq_search": (i32, [P, P, u32, P, u32, u32, u32, P, P, P]),
        "riki_rpq_search_batch": (i32, [P, u32, P, P, P, P, u32, u32, P, P]),
        "riki_rpq_search_batch_device": (i32, [P, u32, P, P, P, P, u32, u32, P]),
        "riki_batch_fetch": (i32, [P, u32, P]),
        "riki_results_count": (u32, [P]),
        "riki_results_get": (i32, [P, u32, P]),
        "riki_results_stats": (i32, [P, P]),
        "riki_results_ncand": (u32, [P]),
        "riki_results_cand": (i32, [P, u32, P, P]),
        "riki_results_free": (None, [P]),
        "riki_results_export_sizes": (i32, [P, u32, P]),
        "riki_results_export": (i32, [P, u32, P, P, P, P, P, P, P, P, P]),
        "riki_hitting_levels": (i32, [P, P, u32, u32, i32, P, P, P, P]),
        "riki_set_profiling": (i32, [P, i32]),
        "riki_get_stats": (i32, [P, P]),
        "riki_reset_stats": (i32, [P]),
        "riki_set_debug": (i32, [P, i32]),
        "riki_set_direction": (i32, [P, i32]),
        "riki_set_joint": (i32, [P, i32]),
        "riki_set_batch_slots": (i32, [P, u32]),
        "riki_memory_footprint": (i32, [P, P, P]),
        "riki_set_arena_limit": (i32, [P, u64]),
        "riki_sample_avg_hops": (i32, [P, u32, P, P, u32, P, P, P, P]),
        "riki_dist_unique_id": (i32, [P]),
        "riki_dist_init": (i32, [P, i32, i32, P, i32]),
        "riki_dist_partition": (i32, [P, u32, u32, P]),
        "riki_dist_info": (i32, [P, P, P, P, P, P, P]),
        "riki_debug_ln_table": (i32, [i32, u64, u64, P]),
        "riki_last_error": (C.c_char_p, []),
        "riki_version": (C.c_char_p, []),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def debug_ln_table(n0: int, count: int, device: int = 0) -> np.ndarray:
    """The device's ln(n) for n in [n0, n0 + count), as the fine-weight kernel computes it
    (riki_debug_ln_table)."""
    out = np.empty(count, np.float64)
    _check(load().riki_debug_ln_table(device, n0, count, _p(out)))
    return out


def dist_unique_id() -> bytes:
    """A fresh 128-byte NCCL unique id (riki_dist_unique_id) for riki_dist_init."""
    buf = C.create_string_buffer(128)
    _check(load().riki_dist_unique_id(buf))
    return buf.raw


def dist_partition(irow, nranks) -> np.ndarray:
    """Vertex-partition bounds for an in-CSR row pointer (host-only, riki_dist_partition)."""
    irow = np.ascontiguousarray(irow, np.uint32)
    b = np.zeros(nranks + 1, np.uint32)
    _check(load().riki_dist_partition(_p(irow), len(irow) - 1, nranks, _p(b)))
    return b


def _check(rc):
    if rc != 0:
        raise RikiError(rc, load().riki_last_error().decode())


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None and a.size else None


def params(gamma=0.5, beam_w=0, beam_mode=0, tie_break=0, ptc_mode=0, early_term=0) -> Params:
    return Params(gamma, beam_w, beam_mode, tie_break, ptc_mode, early_term)


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


@dataclass
class Result:
    rpgs: list
    stats: dict
    candidates: list = field(default_factory=list)  # [(sc, v)] when debug is on


def _take_results(lib, h, nc, nm) -> Result:
    try:
        out = []
        s = RPGStruct()
        for i in range(lib.riki_results_count(h)):
            _check(lib.riki_results_get(h, i, C.byref(s)))
            out.append(RPG(s.central_node, s.sc, s.sm, s.score, s.ptc,
                           np.ctypeslib.as_array(s.nodes, (s.n_nodes,)).copy() if s.n_nodes else np.zeros(0, np.uint32),
                           np.ctypeslib.as_array(s.edge_ids, (s.n_edges,)).copy() if s.n_edges else np.zeros(0, np.uint64),
                           np.ctypeslib.as_array(s.vc, (s.n_vc,)).copy() if s.n_vc else np.zeros(0, np.uint32),
                           np.array([s.cdist[j] for j in range(nc)], np.uint8),
                           np.array([s.mdist[j] for j in range(nm)], np.uint8)))
        qs = QueryStats()
        _check(lib.riki_results_stats(h, C.byref(qs)))
        st = {f: getattr(qs, f) for f, _ in QueryStats._fields_}
        cands = []
        v, sc = C.c_uint32(), C.c_uint32()
        for i in range(lib.riki_results_ncand(h)):
            _check(lib.riki_results_cand(h, i, C.byref(v), C.byref(sc)))
            cands.append((sc.value, v.value))
        return Result(out, st, cands)
    finally:
        lib.riki_results_free(h)


class BatchResult(Sequence):
    """Results of a batch in columnar form (what riki_results_export fills): per-query RPG
    counts, RPG headers / scores and the concatenated node, edge, V_C and distance arrays.
    Behaves as a read-only list of Result; a query's Result is built on first access."""

    def __init__(self, n, ncs, nms, cnt, hdr, score, nodes, edges, vc, cd, md, stats):
        self.n, self.ncs, self.nms = n, ncs, nms
        self.cnt, self.hdr, self.score = cnt, hdr, score
        self.nodes, self.edges, self.vc, self.cd, self.md = nodes, edges, vc, cd, md
        self.stats = stats  # numpy structured array (QueryStats fields)
        self.rpg_off = np.zeros(n + 1, np.int64)
        np.cumsum(cnt, out=self.rpg_off[1:])
        nrpg = int(self.rpg_off[-1])
        self.node_off = np.zeros(nrpg + 1, np.int64)
        self.edge_off = np.zeros(nrpg + 1, np.int64)
        self.vc_off = np.zeros(nrpg + 1, np.int64)
        if nrpg:
            np.cumsum(hdr[:nrpg, 4], out=self.node_off[1:])
            np.cumsum(hdr[:nrpg, 5], out=self.edge_off[1:])
            np.cumsum(hdr[:nrpg, 6], out=self.vc_off[1:])
        self._cache = {}

    def __len__(self):
        return self.n

    def _build(self, i):
        rp = []
        for r in range(int(self.rpg_off[i]), int(self.rpg_off[i + 1])):
            h = self.hdr[r]
            rp.append(RPG(int(h[0]), int(h[1]), int(h[2]), float(self.score[r]), int(h[3]),
                          self.nodes[self.node_off[r]:self.node_off[r + 1]],
                          self.edges[self.edge_off[r]:self.edge_off[r + 1]],
                          self.vc[self.vc_off[r]:self.vc_off[r + 1]],
                          self.cd[r, :self.ncs[i]], self.md[r, :self.nms[i]]))
        st = self.stats[i]
        return Result(rp, {f: int(st[f]) for f in self.stats.dtype.names})

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(self.n))]
        if i < 0:
            i += self.n
        if not 0 <= i < self.n:
            raise IndexError(i)
        if i not in self._cache:
            self._cache[i] = self._build(i)
        return self._cache[i]


def _take_batch(lib, hs, n, ncs, nms) -> BatchResult:
    """Bulk export of n result handles (one C call into preallocated arrays), then free them."""
    try:
        z = ExportSizes()
        _check(lib.riki_results_export_sizes(C.cast(hs, C.c_void_p), n, C.byref(z)))
        cnt = np.zeros(n, np.uint32)
        hdr = np.zeros((max(z.n_rpg, 1), 8), np.uint32)
        score = np.zeros(max(z.n_rpg, 1), np.float64)
        nodes = np.zeros(max(z.n_nodes, 1), np.uint32)
        edges = np.zeros(max(z.n_edges, 1), np.uint64)
        vc = np.zeros(max(z.n_vc, 1), np.uint32)
        cd = np.zeros((max(z.n_rpg, 1), 8), np.uint8)
        md = np.zeros((max(z.n_rpg, 1), 8), np.uint8)
        stats = np.zeros(max(n, 1), dtype=_STATS_DT)
        _check(lib.riki_results_export(C.cast(hs, C.c_void_p), n, _p(cnt), _p(hdr), _p(score), _p(nodes), _p(edges),
                                       _p(vc), _p(cd), _p(md), C.c_void_p(stats.ctypes.data)))
        return BatchResult(n, list(ncs), list(nms), cnt, hdr, score, nodes, edges, vc, cd, md, stats[:n])
    finally:
        for i in range(n):
            lib.riki_results_free(C.c_void_p(hs[i]))


class Graph:
    """Device-resident knowledge graph (riki_load_graph).  Arrays are host numpy arrays."""

    def __init__(self, n_nodes, src, dst, label_class, term_ptr, postings, device=0):
        self.lib = load()
        self.h = None
        src = np.ascontiguousarray(src, np.uint32)
        dst = np.ascontiguousarray(dst, np.uint32)
        cls = np.ascontiguousarray(label_class, np.uint32) if label_class is not None else None
        tp = np.ascontiguousarray(term_ptr, np.uint64)
        po = np.ascontiguousarray(postings, np.uint32)
        h = C.c_void_p()
        _check(self.lib.riki_load_graph(device, int(n_nodes), len(src), _p(src), _p(dst), _p(cls),
                                        len(tp) - 1, _p(tp), _p(po), C.byref(h)))
        self.h = h
        self._debug = False
        self.V = int(n_nodes)
        self.E = len(src)

    @classmethod
    def from_device(cls, n_nodes, n_edges, src_ptr, dst_ptr, cls_ptr, n_terms, tptr_ptr, post_ptr, device=0):
        """riki_load_graph_device: every array a device pointer (int, e.g. tensor.data_ptr());
        u32 src/dst/label_class[n_edges], u64 term_ptr[n_terms + 1], u32 postings."""
        self = cls.__new__(cls)
        self.lib = load()
        self.h = None
        h = C.c_void_p()
        _check(self.lib.riki_load_graph_device(device, int(n_nodes), int(n_edges), C.c_void_p(src_ptr),
                                               C.c_void_p(dst_ptr), C.c_void_p(cls_ptr) if cls_ptr else None,
                                               int(n_terms), C.c_void_p(tptr_ptr), C.c_void_p(post_ptr), C.byref(h)))
        self.h = h
        self._debug = False
        self.V = int(n_nodes)
        self.E = int(n_edges)
        return self

    def close(self):
        if self.h:
            self.lib.riki_free_graph(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- weights
    def set_edge_weights(self, w01, alpha, avg_hops):
        w = np.ascontiguousarray(w01, np.float64)
        _check(self.lib.riki_set_edge_weights(self.h, _p(w), alpha, avg_hops))

    def set_node_weights(self, w01, alpha, avg_hops):
        w = np.ascontiguousarray(w01, np.float64)
        _check(self.lib.riki_set_node_weights(self.h, _p(w), alpha, avg_hops))

    def set_label_weights(self, alpha, avg_hops):
        _check(self.lib.riki_set_label_weights(self.h, alpha, avg_hops))

    def set_activation_levels(self, a):
        a = np.ascontiguousarray(a, np.uint8)
        _check(self.lib.riki_set_activation_levels(self.h, _p(a)))

    def activation_levels(self):
        a = np.zeros(self.E, np.uint8)
        _check(self.lib.riki_get_activation_levels(self.h, _p(a)))
        return a

    # -- debug boundary
    def hitting_levels(self, terms, depth, block_mode):
        t = np.ascontiguousarray(terms, np.uint32)
        H = np.zeros((self.V, len(t)), np.uint8)
        b = np.zeros(self.V, np.uint8)
        rel = C.c_uint64()
        L = C.c_int32()
        _check(self.lib.riki_hitting_levels(self.h, _p(t), len(t), depth, block_mode, _p(H), _p(b), C.byref(rel),
                                            C.byref(L)))
        return H, b, int(rel.value), int(L.value)

    # -- search
    def search(self, central, marginal, k, depth, stream=None, **kw) -> Result:
        """stream: a cudaStream_t handle (e.g. torch.cuda.Stream().cuda_stream) the search is
        issued on, or None for the library stream."""
        c = np.ascontiguousarray(central, np.uint32)
        m = np.ascontiguousarray(marginal, np.uint32)
        prm = params(**kw)
        h = C.c_void_p()
        _check(self.lib.riki_rpq_search(self.h, _p(c), len(c), _p(m), len(m), k, depth, C.byref(prm),
                                        C.c_void_p(stream) if stream else None, C.byref(h)))
        return _take_results(self.lib, h, len(c), len(m))

    @staticmethod
    def _csr(lists):
        ptr = np.zeros(len(lists) + 1, np.uint64)
        ptr[1:] = np.cumsum([len(x) for x in lists])
        flat = np.ascontiguousarray(np.concatenate([np.asarray(x, np.uint32) for x in lists])
                                    if lists else np.zeros(0, np.uint32), np.uint32)
        return ptr, flat

    def search_batch(self, centrals, marginals, k, depth, **kw) -> list:
        cp, ct = self._csr(centrals)
        mp, mt = self._csr(marginals)
        n = len(centrals)
        hs = (C.c_void_p * max(n, 1))()
        prm = params(**kw)
        _check(self.lib.riki_rpq_search_batch(self.h, n, _p(cp), _p(ct), _p(mp), _p(mt), k, depth, C.byref(prm),
                                              C.cast(hs, C.c_void_p)))
        if self._debug:  # candidate lists are only exposed per handle
            return [_take_results(self.lib, C.c_void_p(hs[i]), len(centrals[i]), len(marginals[i]))
                    for i in range(n)]
        return _take_batch(self.lib, hs, n, [len(c) for c in centrals], [len(m) for m in marginals])

    def search_batch_device(self, n, d_cptr, d_cterms, d_mptr, d_mterms, k, depth, **kw):
        """Device pointers (ints, e.g. torch tensor .data_ptr()); results stay on the device."""
        prm = params(**kw)
        _check(self.lib.riki_rpq_search_batch_device(self.h, n, C.c_void_p(d_cptr), C.c_void_p(d_cterms),
                                                     C.c_void_p(d_mptr), C.c_void_p(d_mterms), k, depth,
                                                     C.byref(prm)))

    def fetch(self, n, ncs, nms) -> list:
        hs = (C.c_void_p * max(n, 1))()
        _check(self.lib.riki_batch_fetch(self.h, n, C.cast(hs, C.c_void_p)))
        return _take_batch(self.lib, hs, n, ncs, nms)

    # -- instrumentation
    def set_profiling(self, on=True):
        _check(self.lib.riki_set_profiling(self.h, int(on)))

    def set_debug(self, on=True):
        _check(self.lib.riki_set_debug(self.h, int(on)))
        self._debug = bool(on)

    def set_direction(self, mode):
        """0 = push (default), 1 = direction-optimising (pull for dense frontiers)."""
        _check(self.lib.riki_set_direction(self.h, mode))

    def set_joint(self, on=True):
        """Joint multi-query traversal for large batches (identical results)."""
        _check(self.lib.riki_set_joint(self.h, int(on)))

    def sample_avg_hops(self, src, dst, max_hops=255):
        """Abar from sampled pairs (riki_sample_avg_hops): (mean, sample std, n_reached, dist[])."""
        s_ = np.ascontiguousarray(src, np.uint32)
        t_ = np.ascontiguousarray(dst, np.uint32)
        assert len(s_) == len(t_)
        dist = np.zeros(len(s_), np.uint32)
        m, sd, n = C.c_double(), C.c_double(), C.c_uint64()
        _check(self.lib.riki_sample_avg_hops(self.h, len(s_), _p(s_), _p(t_), int(max_hops), C.byref(m), C.byref(sd),
                                             C.byref(n), _p(dist)))
        return m.value, sd.value, n.value, dist

    def set_arena_limit(self, words):
        _check(self.lib.riki_set_arena_limit(self.h, int(words)))

    def set_batch_slots(self, n):
        _check(self.lib.riki_set_batch_slots(self.h, n))

    def stats(self) -> dict:
        s = Stats()
        _check(self.lib.riki_get_stats(self.h, C.byref(s)))
        d = {f: getattr(s, f) for f, _ in Stats._fields_}
        d["section_ms"] = list(d["section_ms"])
        return d

    def reset_stats(self):
        _check(self.lib.riki_reset_stats(self.h))

    # -- multi-GPU (include/riki.h riki_dist_*)
    def dist_init(self, nranks, rank, unique_id=None, mode=1):
        """mode 1 = vertex-partitioned (unique_id: 128 bytes from dist_unique_id(); None with
        nranks > 1 simulates the nranks partitions in this process), mode 0 = replicated."""
        buf = None
        if unique_id is not None:
            assert len(unique_id) == 128
            buf = C.create_string_buffer(bytes(unique_id), 128)
        _check(self.lib.riki_dist_init(self.h, int(nranks), int(rank), buf, int(mode)))

    def dist_info(self) -> dict:
        n, r, m = C.c_int(), C.c_int(), C.c_int()
        _check(self.lib.riki_dist_info(self.h, C.byref(n), C.byref(r), C.byref(m), None, None, None))
        b = np.zeros(n.value + 1, np.uint32)
        x, xb = C.c_uint64(), C.c_uint64()
        _check(self.lib.riki_dist_info(self.h, None, None, None, _p(b), C.byref(x), C.byref(xb)))
        return {"nranks": n.value, "rank": r.value, "mode": m.value, "bounds": b, "exchanges": x.value,
                "exchanged_bytes": xb.value}

    def memory_footprint(self):
        a, b = C.c_uint64(), C.c_uint64()
        _check(self.lib.riki_memory_footprint(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value
