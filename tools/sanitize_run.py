"""Small workloads through every kernel family, for compute-sanitizer (memcheck/racecheck/synccheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2001_06770_b200 as P
import synth
kg = synth.make_kg(1)
qs = synth.config_queries(kg, 1, 40)
g = P.Graph(kg.n_nodes, kg.src, kg.dst, kg.label_class, kg.term_ptr, kg.postings)
g.set_label_weights(0.5, kg.avg_hops)
g.set_debug(True)
n = 0
for mode in range(3):
    H, b, rel, L = g.hitting_levels(np.arange(4, dtype=np.uint32), 20, mode)
for joint in (0, 1):
    g.set_joint(joint)
    for kw in (dict(), dict(ptc_mode=1), dict(ptc_mode=2, early_term=1), dict(ptc_mode=3, early_term=2, beam_mode=1)):
        res = g.search_batch(qs.central, qs.marginal, qs.k, 20, **kw)
        n += sum(len(r.rpgs) for r in res)
g.set_joint(0)
g.set_direction(1)
res = g.search_batch(qs.central, qs.marginal, qs.k, 20)
g.set_direction(0)
for i in range(3):
    g.search(qs.central[i], qs.marginal[i], qs.k, 20)
print("sanitize workload done, rpgs", n)
