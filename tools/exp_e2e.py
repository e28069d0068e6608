"""Where the end-to-end time goes (config 2 batch): device-resident call vs host call, and the
host call split into the C batch search and the Python-side export."""
import ctypes as C
import gc
import time

import numpy as np
import torch

import paper_2001_06770_b200 as P
from paper_2001_06770_b200 import riki as R
import synth

kg = synth.make_kg(2)
qs = synth.config_queries(kg, 2, 200)
g = P.Graph(kg.n_nodes, kg.src, kg.dst, kg.label_class, kg.term_ptr, kg.postings)
g.set_label_weights(0.5, kg.avg_hops)
g.set_batch_slots(200)
cp, ct = P.Graph._csr(qs.central)
mp, mt = P.Graph._csr(qs.marginal)
d = [torch.from_numpy(x.view(np.int64) if x.dtype == np.uint64 else x.view(np.int32)).cuda() for x in (cp, ct, mp, mt)]
for _ in range(3):
    g.search_batch(qs.central, qs.marginal, qs.k, qs.depth)
gc.collect(); gc.disable()
def t(fn, n=10):
    ts = []
    for _ in range(n):
        torch.cuda.synchronize(); a = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - a)
    return 1e3 * float(np.median(ts))
dev = t(lambda: g.search_batch_device(200, *[x.data_ptr() for x in d], qs.k, qs.depth))
host = t(lambda: g.search_batch(qs.central, qs.marginal, qs.k, qs.depth))
n = 200
hs = (C.c_void_p * n)()
prm = R.params()
def c_only():
    R._check(g.lib.riki_rpq_search_batch(g.h, n, R._p(cp), R._p(ct), R._p(mp), R._p(mt), qs.k, qs.depth, C.byref(prm),
                                         C.cast(hs, C.c_void_p)))
ts_c, ts_x = [], []
for _ in range(10):
    a = time.perf_counter(); c_only(); b = time.perf_counter()
    R._take_batch(g.lib, hs, n, [2] * n, [2] * n); e = time.perf_counter()
    ts_c.append(b - a); ts_x.append(e - b)
print(f"device call {dev:.2f} ms | host call {host:.2f} ms | C batch {1e3*np.median(ts_c):.2f} ms | export {1e3*np.median(ts_x):.2f} ms")
g.set_profiling(True); g.reset_stats()
g.search_batch(qs.central, qs.marginal, qs.k, qs.depth)
print("sections (host wall between syncs):", g.stats()["section_ms"])
