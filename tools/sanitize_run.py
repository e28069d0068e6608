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
        print("step joint", joint, kw, flush=True)
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
# bounded RPG recovery (k_rpg_select waves), forced on the small config
os.environ["RIKI_BOUNDED_RPG"] = "1"
res = g.search_batch(qs.central, qs.marginal, qs.k, 20, ptc_mode=1)
del os.environ["RIKI_BOUNDED_RPG"]
# row-width groups: a batch mixing 1-8 keywords per run
mix_c = [qs.central[i][:1 + i % 2] for i in range(len(qs.central))]
mix_m = [(qs.marginal[i] + qs.central[i])[: (i % 4) * 2] for i in range(len(qs.central))]
res = g.search_batch(mix_c, mix_m, qs.k, 20)
# the coarsening's ln table (R31)
P.riki.debug_ln_table(1, 1 << 20)
# vertex-partitioned push (k_expand / k_expand_heavy VPX, k_vp_apply_words): 3 simulated partitions
g.dist_init(3, 0, None, mode=1)
for mode in range(3):
    g.hitting_levels(np.arange(4, dtype=np.uint32), 20, mode)
res = g.search_batch(qs.central, qs.marginal, qs.k, 20)
n += sum(len(r.rpgs) for r in res)
# ... and the pull variant (k_pull ranges, k_vp_apply)
os.environ["RIKI_VP_PULL"] = "1"
g.dist_init(2, 0, None, mode=1)
res = g.search_batch(qs.central, qs.marginal, qs.k, 20)
del os.environ["RIKI_VP_PULL"]
n += sum(len(r.rpgs) for r in res)
print("sanitize workload done, rpgs", n)
