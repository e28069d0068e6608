"""Experiment: does overlapping two independent half-batches (two graph handles = two
workspaces and library streams, two host threads) beat one lock-step batch on config 2?"""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2001_06770_b200 as P
import synth

kg = synth.make_kg(2)
qs = synth.config_queries(kg, 2)
nq = len(qs.central)


def dev_arrays(lo, hi):
    cp, ct = P.Graph._csr(qs.central[lo:hi])
    mp, mt = P.Graph._csr(qs.marginal[lo:hi])
    return [torch.from_numpy(x.view(np.int64) if x.dtype == np.uint64 else x.view(np.int32)).cuda()
            for x in (cp, ct, mp, mt)]


for nsplit in (1, 2, 3, 4):
    gs, arrs, ns = [], [], []
    for i in range(nsplit):
        lo, hi = i * nq // nsplit, (i + 1) * nq // nsplit
        g = P.Graph(kg.n_nodes, kg.src, kg.dst, kg.label_class, kg.term_ptr, kg.postings)
        g.set_label_weights(0.5, kg.avg_hops)
        g.set_batch_slots(hi - lo)
        gs.append(g)
        arrs.append(dev_arrays(lo, hi))
        ns.append(hi - lo)

    def run(i):
        gs[i].search_batch_device(ns[i], *(x.data_ptr() for x in arrs[i]), qs.k, qs.depth)

    def step():
        ts = [threading.Thread(target=run, args=(i,)) for i in range(nsplit)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        step()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 10
    print(f"{nsplit} concurrent sub-batches: {dt * 1e3:.2f} ms per 200-query step = {nq / dt:.0f} q/s", flush=True)
    del gs, arrs
    torch.cuda.empty_cache()
