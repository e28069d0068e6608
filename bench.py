"""Benchmark of the RIKI hot path on B200.

python bench.py [--gpus N --steps K --warmup W] [--impl riki|reference] [--config 2]

A step = one batch of the config's synthetic RPQ workload (config 2: 200 queries, 2 central +
2 marginal keywords, k = 10, depth 20, on a 1M-node / 5M-edge power-law KG) through the
whole hot path (both runs, recovery, PTC, top-k) with inputs resident in HBM.  Under
torchrun every rank runs its own batch on its own GPU (query-sharded replicas, weak
scaling, no collective on the data path); the time is the max over ranks.
--impl reference times the CPU oracle (oracle/, the only reference this paper has) on a
bounded sample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "RPQ queries/sec"
UNIT = "queries/s"


def _workload_name(cfg, spec):
    if cfg == 5:
        return (f"C5 {spec.name}: config 4's synthetic KG ({spec.n_nodes} nodes / {spec.n_edges} directed edges), "
                f"batch of {spec.n_queries} queries: half 2 central + 4 marginal, half the Exp-1 mix "
                f"{{1,2,4}} x {{2,4,6}}, k={spec.k}, depth {spec.depth}")
    return (f"C{cfg} {spec.name}: synthetic power-law KG {spec.n_nodes} nodes / {spec.n_edges} directed edges, "
            f"{spec.n_central} central + {spec.n_marginal} marginal keywords, k={spec.k}, depth {spec.depth}")


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 8:
                continue
            try:
                sm.append(float(p[0]))
                mx = max(mx, float(p[1]))
            except ValueError:
                continue
            for n, v in zip(names, p[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws <= 1:
        return 0, 1, None
    import torch
    import torch.distributed as dist
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    # RIKI_BENCH_BACKEND=gloo lets several ranks share one GPU (tests of the multi-rank path);
    # the contract run uses NCCL, one process per GPU
    backend = os.environ.get("RIKI_BENCH_BACKEND", "nccl")
    torch.cuda.set_device(local % torch.cuda.device_count())
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    return rank, ws, dist


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def oracle_sample(kg, qs, idx, og=None, threads=1):
    """Times the CPU oracle (as it stands) on queries idx, one query per thread on `threads`
    host threads (the oracle is plain C behind ctypes, which releases the GIL, and keeps no
    global state); returns (seconds, og)."""
    import oracle as O
    if og is None:
        w = O.fine_weights(kg.n_nodes, kg.src, kg.dst, kg.label_class)
        og = O.Graph(kg.n_nodes, kg.src, kg.dst, O.coarsen_all(w, 0.5, kg.avg_hops))

    def one(i):
        O.search(og, [kg.posting(t) for t in qs.central[i]], [kg.posting(t) for t in qs.marginal[i]], qs.k,
                 qs.depth, want_matrices=False, want_candidates=False)

    t0 = time.perf_counter()
    if threads <= 1:
        for i in idx:
            one(i)
    else:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(one, idx))
    return time.perf_counter() - t0, og


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import synth
    spec = synth.CONFIGS[args.config]
    kg = synth.make_kg(args.config)
    qs = synth.config_queries(kg, args.config)
    cores = host_cores()
    per = args.ref_queries or min(len(qs.central), 2 * cores)
    og = None
    for s in range(args.warmup):
        _, og = oracle_sample(kg, qs, [(s * per + j) % len(qs.central) for j in range(per)], og, cores)
    times = []
    for s in range(args.steps):
        i0 = ((args.warmup + s) * per) % len(qs.central)
        dt, og = oracle_sample(kg, qs, [(i0 + j) % len(qs.central) for j in range(per)], og, cores)
        times.append(dt)
    tot = sum(times)
    v = per * args.steps / tot
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": _workload_name(args.config, spec), "queries_per_step": per},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{per} queries of the config-{args.config} query set per step, "
                                       f"oracle/riki_oracle.c, one query per thread on {cores} host cores"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="riki", choices=["riki", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--queries", type=int, default=0, help="queries per step (default: the config's query set)")
    ap.add_argument("--cpu-sample", type=int, default=16, help="oracle queries for cpu_baseline")
    ap.add_argument("--ref-queries", type=int, default=0,
                    help="oracle queries per step for --impl reference (0 = 2 per host core)")
    ap.add_argument("--latency-queries", type=int, default=40)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--quick", action="store_true", help="timed region only (for ncu launch lists)")
    ap.add_argument("--slots", type=int, default=0, help="queries in flight per launch (0 = whole batch)")
    ap.add_argument("--pull", action="store_true", help="enable the direction-optimising (pull) expansion")
    ap.add_argument("--joint", type=int, default=0, help="1 = joint multi-query traversal for the batch")
    ap.add_argument("--vp", action="store_true",
                    help="vertex-partitioned mode (SURVEY §8(e)): every rank runs the SAME batch, each pulling "
                         "its node range, one NCCL all-gather of frontier bit planes per level (strong scaling)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
        return

    import torch

    import paper_2001_06770_b200 as P
    import synth
    from paper_2001_06770_b200.dist import gather_results, max_over_ranks

    rank, world, dist = _dist()
    dev = torch.cuda.current_device()
    spec = synth.CONFIGS[args.config]
    kg = synth.make_kg(args.config)
    nq = args.queries or spec.n_queries
    if world == 1 or args.vp:
        qs = synth.config_queries(kg, args.config, nq)
    elif args.config == 5:  # weak scaling: each rank its own batch of the same mix
        qs = synth.c5_queries(kg, nq, 2005 + 7919 * rank)
    else:  # weak scaling: each rank its own query batch of the same shape
        qs = synth.make_queries(kg, nq, spec.n_central, spec.n_marginal, spec.k, spec.depth,
                                2000 + args.config + 7919 * rank)
    g = P.Graph(kg.n_nodes, kg.src, kg.dst, kg.label_class, kg.term_ptr, kg.postings, device=dev)
    g.set_label_weights(0.5, kg.avg_hops)
    g.set_batch_slots(args.slots or min(nq, 1024))
    g.set_direction(1 if args.pull else 0)
    g.set_joint(bool(args.joint))
    if args.vp:
        if dist:
            from paper_2001_06770_b200.dist import init_vertex_partitioned
            init_vertex_partitioned(g)
        else:
            g.dist_init(1, 0, P.riki.dist_unique_id(), mode=1)
    units = 1 if args.vp else world  # VP: all ranks cooperate on one batch
    cp, ct = P.Graph._csr(qs.central)
    mp, mt = P.Graph._csr(qs.marginal)
    d_cp, d_ct, d_mp, d_mt = [torch.from_numpy(x.view(np.int64) if x.dtype == np.uint64 else x.view(np.int32))
                              .to(f"cuda:{dev}") for x in (cp, ct, mp, mt)]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev}")  # > 126 MB L2

    def step_device():
        g.search_batch_device(nq, d_cp.data_ptr(), d_ct.data_ptr(), d_mp.data_ptr(), d_mt.data_ptr(), qs.k, qs.depth)

    def barrier():
        if dist:
            dist.barrier()

    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()
    gc.collect()   # no Python GC pauses inside timed regions
    gc.disable()
    # ---------------- timed region (device-resident inputs and results)
    g.reset_stats()
    g.set_profiling(True)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    with Clocks(dev) as clk:
        for i in range(args.steps):
            flush.fill_(i & 0xFF)      # L2 flush, finished before the step starts (the library
            torch.cuda.synchronize()   # runs on its own stream and would overlap with it)
            ev[i][0].record()
            step_device()
            ev[i][1].record()
        torch.cuda.synchronize()
    barrier()
    g.set_profiling(False)
    st = g.stats()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    tot_ms = sum(step_ms)
    rdev = f"cuda:{dev}" if not dist or dist.get_backend() == "nccl" else None
    tot_ms = max_over_ranks(tot_ms, device=rdev)  # time = slowest rank (weak scaling)
    value = nq * units * args.steps / (tot_ms / 1000.0)
    res = g.fetch(nq, [len(c) for c in qs.central], [len(m) for m in qs.marginal])
    relax = sum(r.stats["relax_central"] + r.stats["relax_marginal"] for r in res)
    n_rpg = sum(len(r.rpgs) for r in res)

    if args.quick:
        if rank == 0:
            print(json.dumps({"metric": METRIC, "value": value, "unit": UNIT, "ms_per_step": tot_ms / args.steps,
                              "quick": True, "stats": st}), flush=True)
        return
    # ---------------- e2e through the host C-ABI (H2D of queries, D2H of results inside)
    h2d = cp.nbytes + ct.nbytes + mp.nbytes + mt.nbytes
    e2e_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    torch.cuda.synchronize()
    d2h = 0
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        torch.cuda.synchronize()
        e2e_ev[i][0].record()
        rr = g.search_batch(qs.central, qs.marginal, qs.k, qs.depth)
        if dist and not args.vp:  # replicated mode: every shard's results gathered to rank 0
            gather_results(rr, device=rdev)
        e2e_ev[i][1].record()
        d2h = sum(4 * (len(x.nodes) + len(x.vc)) + 4 * len(x.edge_ids) + 64 for r in rr for x in r.rpgs)
    torch.cuda.synchronize()
    barrier()
    e2e_ms = sum(a.elapsed_time(b) for a, b in e2e_ev)
    e2e_ms = max_over_ranks(e2e_ms, device=rdev)
    e2e_value = nq * units * args.steps / (e2e_ms / 1000.0)

    # ---------------- single-query latency (one query in flight, host API incl. D2H)
    del rr
    gc.collect()
    for i in range(3):  # warm the single-slot path
        g.search(qs.central[i], qs.marginal[i], qs.k, qs.depth)
    lat = []
    for i in range(min(args.latency_queries, nq)):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.search(qs.central[i], qs.marginal[i], qs.k, qs.depth)
        b.record()
        torch.cuda.synchronize()
        lat.append(a.elapsed_time(b))
    lat.sort()
    gc.enable()

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    peak, peak_src = _peaks()
    traffic, traffic_src = None, None
    try:  # DRAM bytes of the expansion launches from the committed ncu capture (profiles/)
        import glob
        tf = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_expand_traffic.json")))[-1]
        tj = json.load(open(tf))
        traffic = tj["dram_bytes_per_launch"]
        traffic_src = f"{os.path.relpath(tf, ROOT)}: {tj['dram_bytes_step'] / 1e9:.2f} GB DRAM vs " \
                      f"{(tj['algorithmic_bytes_step'] or 0) / 1e9:.2f} GB algorithmic per step"
    except Exception:
        pass
    achieved = (st["expand_bytes"] / 1e9) / (st["expand_ms"] / 1e3) if st["expand_ms"] > 0 else 0.0
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": tot_ms / args.steps, "higher_is_better": True, "scaling": "strong" if args.vp else "weak",
        "vs_baseline": None,
        "dtype": "u8", "data": "synthetic",
        "config": {"workload": _workload_name(args.config, spec), "queries_per_step_per_gpu": nq,
                   "l2": "flushed between steps (256 MiB write)", "parallelism": f"vertex-partitioned x{world} (NCCL bit-plane all-gather per level)" if args.vp
                   else f"query-sharded replicas x{world}",
                   "graph_seed": 1000 + synth.GRAPH_OF.get(args.config, args.config), "query_seed": 2000 + args.config},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak if peak else None, "traffic": traffic, "traffic_source": traffic_src,
                     "achieved_bytes_per_launch": st["expand_bytes"] / max(1, st["expand_launches"]),
                     "kernel": "k_expand + k_expand_heavy (Alg. 1 expansion), CUDA events on the library stream",
                     "sections_ms_per_step": [x / args.steps for x in st["section_ms"]], "levels_per_step": st["levels"] / args.steps,
                     "peak_source": peak_src, "expand_share_of_step": st["expand_ms"] / tot_ms if tot_ms else None},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "results_gathered_to_rank0": bool(dist) and not args.vp},
        "gpu_launches": int(st["kernel_launches"]),
        "latency_ms": {"p50": lat[len(lat) // 2] if lat else None,
                       "p99": lat[min(len(lat) - 1, int(0.99 * len(lat)))] if lat else None, "n": len(lat)},
        "gteps": relax / (tot_ms / args.steps / 1000.0) / 1e9,
        "relaxations_per_step": relax, "rpgs_per_step": n_rpg,
        "step_ms": [round(x, 3) for x in step_ms],
        "clocks": clk.summary(),
    }
    if args.vp:
        di = g.dist_info()
        line["vp"] = {"nranks": di["nranks"], "bounds": di["bounds"].tolist(), "exchanges": di["exchanges"],
                      "exchanged_bytes": di["exchanged_bytes"]}
    if world == 1 and not args.no_cpu:
        cores = host_cores()
        n1 = min(args.cpu_sample, nq)
        dt1, og = oracle_sample(kg, qs, range(n1))
        n = min(max(args.cpu_sample, 2 * cores), nq)
        dt, _ = oracle_sample(kg, qs, range(n), og, cores)
        line["cpu_baseline"] = {"value": n / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
                                "sample": f"first {n} queries of the same batch, one query per thread on {cores} "
                                          f"host cores (oracle as it stands)",
                                "single_core": {"value": n1 / dt1, "cores": 1, "sample": f"first {n1} queries"}}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
