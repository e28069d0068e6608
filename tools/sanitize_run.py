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
# weight-sum tie-break (k_tie_weights / k_tie_select), with the beam truncated by W(CG) (k_beam_tie)
for kw in (dict(tie_break=1), dict(tie_break=1, beam_mode=1, beam_w=qs.k + 1), dict(tie_break=1, ptc_mode=1)):
    res = g.search_batch(qs.central, qs.marginal, qs.k, 20, **kw)
    n += sum(len(r.rpgs) for r in res)
res = g.search_batch(qs.central, [[] for _ in qs.central], qs.k, 20, tie_break=1)  # M empty
# 64-bit frontier-item loop
os.environ["RIKI_FORCE_WIDE"] = "1"
g.search_batch(qs.central, qs.marginal, qs.k, 20)
del os.environ["RIKI_FORCE_WIDE"]
# arena-limit chunking (fresh graph: a small arena)
g2 = P.Graph(kg.n_nodes, kg.src, kg.dst, kg.label_class, kg.term_ptr, kg.postings)
g2.set_label_weights(0.5, kg.avg_hops)
g2.set_arena_limit(1 << 14)
g2.search_batch(qs.central, qs.marginal, qs.k, 20)
# vertex-partitioned mode: 3 simulated partitions (k_pull ranges, k_vp_apply), then 1-rank NCCL
g.dist_init(3, 0, None, mode=1)
for mode in range(3):
    g.hitting_levels(np.arange(4, dtype=np.uint32), 20, mode)
res = g.search_batch(qs.central, qs.marginal, qs.k, 20)
n += sum(len(r.rpgs) for r in res)
print("sanitize workload done, rpgs", n)
