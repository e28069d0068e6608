"""Abar from 10k sampled pairs on the GPU (riki_sample_avg_hops) for configs 2 and 4,
with the time, against the oracle's value on the first 32 pairs.  usage: abar_sample.py [cfg...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle as O
import paper_2001_06770_b200 as P
import synth

for cfg in [int(x) for x in sys.argv[1:]] or [2]:
    kg = synth.make_kg(cfg)
    g = P.Graph(kg.n_nodes, kg.src, kg.dst, kg.label_class, kg.term_ptr, kg.postings)
    rng = np.random.default_rng(611 + cfg)
    ps = rng.integers(0, kg.n_nodes, 10000).astype(np.uint32)
    pt = rng.integers(0, kg.n_nodes, 10000).astype(np.uint32)
    g.sample_avg_hops(ps[:64], pt[:64])  # warm-up
    torch.cuda.synchronize()
    t = time.perf_counter()
    m, sd, n, d = g.sample_avg_hops(ps, pt)
    dt = time.perf_counter() - t
    to = time.perf_counter()
    mo, sdo, no, do = O.sample_avg_hops(kg.n_nodes, kg.src, kg.dst, ps[:32], pt[:32])
    dto = time.perf_counter() - to
    assert (d[:32] == do).all()
    print(f"config {cfg}: V={kg.n_nodes} E={len(kg.src)}: 10k pairs -> Abar {m:.4f} (sd {sd:.4f}, {n} reached) "
          f"in {dt * 1e3:.1f} ms on the GPU; oracle (scipy BFS) {dto:.2f} s for 32 pairs, identical distances; "
          f"the config's Abar input is {kg.avg_hops}", flush=True)
