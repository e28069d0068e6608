"""SURVEY §8(f) f2 / the paper's Exp-2: top-k and beam-variant sweep on config 2.

For k in {5, 10, 20, 40} and the beam variants
  ties   beam_mode 0: every CG identified by the terminating level (R13, default)
  trunc  beam_mode 1: the first w = k CGs by (S^c, v)
  wide   beam_mode 0 with an explicit beam w = 2k
  lit    beam_mode 0 with the paper's literal early-termination inequality (early_term 1)
  tie    beam_mode 0 with the weight-sum tie-break (R29)
it times the 200-query batch on the device (CUDA events, L2 flushed, 3 warm-up + 5 timed
steps) and reports q/s, the central / recovery / marginal section times, the mean number
of candidate CGs and the mean marginal terminating level.  R13's claim to check: with ties
kept, the marginal run's time falls as k grows (more candidates attach early, the exact
bound fires sooner) while the candidate count, not k, drives the recovery time.
usage (GPU box):  python tools/exp2_beam_sweep.py > profiles/<round>_exp2_beam_sweep.txt"""
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
g.set_label_weights(0.5, kg.avg_hops)
g.set_batch_slots(nq)
cp, ct = P.Graph._csr(qs.central)
mp, mt = P.Graph._csr(qs.marginal)
d = [torch.from_numpy(x.view(np.int64) if x.dtype == np.uint64 else x.view(np.int32)).cuda() for x in (cp, ct, mp, mt)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
VARIANTS = {
    "ties": lambda k: dict(),
    "trunc": lambda k: dict(beam_mode=1),
    "wide": lambda k: dict(beam_w=2 * k),
    "lit": lambda k: dict(early_term=1),
    "tie": lambda k: dict(tie_break=1),
}
print(f"# config 2, {nq} queries per step, depth {qs.depth}; 3 warm-up + 5 timed steps per setting")
print(f"# {'k':>3} {'variant':7} {'q/s':>9} {'central_ms':>10} {'recov_ms':>9} {'marg_ms':>8} {'cands':>8} {'Lm':>5} {'rpgs':>6}")
for k in (5, 10, 20, 40):
    for name, kw in VARIANTS.items():
        args = kw(k)

        def step():
            g.search_batch_device(nq, *(x.data_ptr() for x in d), k, qs.depth, **args)

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
        cands = np.mean([r.stats["n_candidates"] for r in res])
        lm = np.mean([r.stats["L_marginal"] for r in res])
        rpgs = np.mean([len(r.rpgs) for r in res])
        sec = [x / 5 for x in st["section_ms"]]
        print(f"  {k:3d} {name:7} {nq * 5 / (sum(ms) / 1e3):9.1f} {sec[0]:10.2f} {sec[1]:9.2f} {sec[2]:8.2f} "
              f"{cands:8.1f} {lm:5.2f} {rpgs:6.2f}", flush=True)
