"""Experiment: effect of queries-in-flight (slots) on the expansion time (host API path)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2001_06770_b200 as P
import synth
kg = synth.make_kg(2)
qs = synth.config_queries(kg, 2)
for S in [int(x) for x in sys.argv[1:]]:
    g = P.Graph(kg.n_nodes, kg.src, kg.dst, kg.label_class, kg.term_ptr, kg.postings)
    g.set_label_weights(0.5, kg.avg_hops)
    g.set_batch_slots(S)
    g.search_batch(qs.central, qs.marginal, qs.k, qs.depth)  # warm + allocate
    g.reset_stats(); g.set_profiling(True)
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(3):
        g.search_batch(qs.central, qs.marginal, qs.k, qs.depth)
    torch.cuda.synchronize(); dt = (time.perf_counter() - t) / 3
    st = g.stats(); g.set_profiling(False)
    g.close()
    print(f"slots {S:4d}: {200/dt:8.0f} q/s  step {1000*dt:6.2f} ms  expand {st['expand_ms']/3:6.2f} ms  sections {[round(x/3,2) for x in st['section_ms']]} levels {st['levels']/3}")
