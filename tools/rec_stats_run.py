"""Run three config-2 batches; with libriki built -DREC_STATS=1 (RIKI_LIB) it prints the recovery
diagnostics line ([riki-rec]: list builds, waits, per-candidate cycle histogram)."""
import sys, os
sys.path.insert(0, os.getcwd())
import paper_2001_06770_b200 as P, synth
kg = synth.make_kg(2); qs = synth.config_queries(kg, 2, 200)
g = P.Graph(kg.n_nodes, kg.src, kg.dst, kg.label_class, kg.term_ptr, kg.postings)
g.set_label_weights(0.5, kg.avg_hops); g.set_batch_slots(200)
for _ in range(3):
    g.search_batch(qs.central, qs.marginal, qs.k, qs.depth)
