"""Bench-like sequence: device batch, host batches, then single queries with per-query stats."""
import sys, os, time, gc
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2001_06770_b200 as P
import synth
kg = synth.make_kg(2)
qs = synth.config_queries(kg, 2)
g = P.Graph(kg.n_nodes, kg.src, kg.dst, kg.label_class, kg.term_ptr, kg.postings)
g.set_label_weights(0.5, kg.avg_hops)
g.set_batch_slots(200)
cp, ct = P.Graph._csr(qs.central); mp, mt = P.Graph._csr(qs.marginal)
d = [torch.from_numpy(x.view(np.int64) if x.dtype == np.uint64 else x.view(np.int32)).cuda() for x in (cp, ct, mp, mt)]
for _ in range(3):
    g.search_batch_device(200, d[0].data_ptr(), d[1].data_ptr(), d[2].data_ptr(), d[3].data_ptr(), qs.k, qs.depth)
for _ in range(3):
    rr = g.search_batch(qs.central, qs.marginal, qs.k, qs.depth)
del rr; gc.collect(); gc.disable()
for i in range(40):
    g.reset_stats(); g.set_profiling(True)
    torch.cuda.synchronize(); t = time.perf_counter()
    r = g.search(qs.central[i], qs.marginal[i], qs.k, qs.depth)
    dt = 1000 * (time.perf_counter() - t)
    st = g.stats(); g.set_profiling(False)
    if dt > 3 or i < 2:
        print(f"q{i}: {dt:.2f} ms retries {st['retries']} reallocs {st['reallocs']} levels {st['levels']} sections {[round(x,2) for x in st['section_ms']]} cands {r.stats['n_candidates']}")
