"""SURVEY §8(f) f4 / the paper's Exp-4: the effect of the coarsening parameter alpha.

For alpha in {0.1, 0.3, 0.5, 0.7, 0.9} the config-2 graph is re-weighted on the GPU
(riki_set_label_weights: label-class fine weights, Eq. 1-3) and the 200-query batch is timed
on the device (CUDA events, L2 flushed, 3 warm-up + 5 timed steps).  Reported: q/s, the
section times, the activation histogram mean, the mean terminating levels of both runs and
the mean relaxation count.  The paper: a small alpha rewards fewer edges, so the search
"stalls" until the global level catches up with the activation levels.
usage (GPU box):  python tools/exp4_alpha_sweep.py > profiles/<round>_exp4_alpha_sweep.txt"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2001_06770_b200 as P
import synth

kg = synth.make_kg(2)
qs = synth.config_queries(kg, 2)
nq = len(qs.central)
g = P.Graph(kg.n_nodes, kg.src, kg.dst, kg.label_class, kg.term_ptr, kg.postings)
g.set_batch_slots(nq)
cp, ct = P.Graph._csr(qs.central)
mp, mt = P.Graph._csr(qs.marginal)
d = [torch.from_numpy(x.view(np.int64) if x.dtype == np.uint64 else x.view(np.int32)).cuda() for x in (cp, ct, mp, mt)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
print(f"# config 2, {nq} queries per step, k={qs.k}, depth {qs.depth}, Abar={kg.avg_hops}; 3 warm-up + 5 timed steps")
print(f"# {'alpha':>5} {'q/s':>9} {'central_ms':>10} {'recov_ms':>9} {'marg_ms':>8} {'mean_a':>7} {'a=0':>6} "
      f"{'Lc':>5} {'Lm':>5} {'relax/q':>10} {'rpgs':>5}")
for alpha in (0.1, 0.3, 0.5, 0.7, 0.9):
    g.set_label_weights(alpha, kg.avg_hops)
    act = g.activation_levels()

    def step():
        g.search_batch_device(nq, *(x.data_ptr() for x in d), qs.k, qs.depth)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    g.reset_stats()
    g.set_profiling(True)
    ms = []
    for i in range(5):
        flush.fill_(i)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        step()
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    st = g.stats()
    g.set_profiling(False)
    res = g.fetch(nq, [len(c) for c in qs.central], [len(m) for m in qs.marginal])
    lc = np.mean([r.stats["L_central"] for r in res])
    lm = np.mean([r.stats["L_marginal"] for r in res])
    rel = np.mean([r.stats["relax_central"] + r.stats["relax_marginal"] for r in res])
    rpgs = np.mean([len(r.rpgs) for r in res])
    sec = [x / 5 for x in st["section_ms"]]
    print(f"  {alpha:5.1f} {nq * 5 / (sum(ms) / 1e3):9.1f} {sec[0]:10.2f} {sec[1]:9.2f} {sec[2]:8.2f} "
          f"{act.mean():7.2f} {np.mean(act == 0):6.1%} {lc:5.2f} {lm:5.2f} {rel:10.0f} {rpgs:5.2f}", flush=True)
