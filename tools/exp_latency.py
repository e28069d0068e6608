"""Single-query latency breakdown (host API, one query in flight)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2001_06770_b200 as P
import synth
kg = synth.make_kg(2)
qs = synth.config_queries(kg, 2)
g = P.Graph(kg.n_nodes, kg.src, kg.dst, kg.label_class, kg.term_ptr, kg.postings)
g.set_label_weights(0.5, kg.avg_hops)
if len(sys.argv) > 1:
    g.set_batch_slots(int(sys.argv[1]))
    g.search_batch(qs.central, qs.marginal, qs.k, qs.depth)
for rep in range(2):
    lat = []
    for i in range(40):
        g.reset_stats(); g.set_profiling(True)
        torch.cuda.synchronize(); t = time.perf_counter()
        r = g.search(qs.central[i], qs.marginal[i], qs.k, qs.depth)
        dt = 1000 * (time.perf_counter() - t)
        st = g.stats(); g.set_profiling(False)
        lat.append(dt)
        if rep == 1 and (dt > 4 or i < 3):
            print(f"q{i}: {dt:.2f} ms retries {st['retries']} reallocs {st['reallocs']} levels {st['levels']} sections {[round(x,2) for x in st['section_ms']]} cands {r.stats['n_candidates']} Lc {r.stats['L_central']} Lm {r.stats['L_marginal']}")
    lat.sort()
    print('p50', round(lat[20], 2), 'p90', round(lat[36], 2), 'max', round(lat[-1], 2))
