"""Benchmark of the RIKI hot path on B200.

python bench.py [--gpus N --steps K --warmup W] [--impl riki|reference] [--config 5]

Default workload: config 5, the largest single-GPU configuration of BASELINE.json -- the
Wikidata-scale synthetic KG (30M nodes / 150M directed edges, WikiLarge-shaped) with
the 10k-query throughput set (half 2 central + 4 marginal, half the Exp-1 mix
{1,2,4} x {2,4,6}; k = 20, depth 20).  A step = one 1,000-query chunk of that set
(step i takes chunk i mod 10, so 10 steps cover all 10k queries) through the whole hot path
(both runs, recovery, attach, PTC, top-k) with inputs resident in HBM, on the production
path (CUDA-graph level loops, no profiling syncs).  A separate profiling pass over the same
chunks measures the expansion kernel's launches with CUDA events (the roofline numbers).
Under torchrun every rank runs its own chunks on its own GPU (query-sharded replicas, weak
scaling, no collective on the data path); the time is the max over ranks.
The oracle (oracle/, the only reference this paper has) is timed on the host cores on a
bounded sample of chunk 0, and its results on that sample gate the GPU line (``parity``).
--impl reference times the oracle alone, on the same workload.
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


def _workload_name(cfg, spec, per_step=None):
    if cfg == 5:
        return (f"C5 {spec.name}: config 4's synthetic KG ({spec.n_nodes} nodes / {spec.n_edges} directed edges), "
                f"{spec.n_queries}-query set: half 2 central + 4 marginal, half the Exp-1 mix "
                f"{{1,2,4}} x {{2,4,6}}, k={spec.k}, depth {spec.depth}; {per_step or spec.n_queries} queries per step")
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


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ---------------------------------------------------------------------------------- oracle side
def oracle_graph(kg):
    """The oracle's own graph: activations from its own fine weights and coarsening (Eq. 1-3)."""
    import oracle as O
    w = O.fine_weights(kg.n_nodes, kg.src, kg.dst, kg.label_class)
    return O.Graph(kg.n_nodes, kg.src, kg.dst, O.coarsen_all(w, 0.5, kg.avg_hops))


def oracle_run(kg, og, qs, idx, threads=1):
    """Runs the CPU oracle (as it stands) on queries idx, one query per thread on `threads`
    host threads (plain C behind ctypes, which releases the GIL).  Returns (wall seconds,
    {query index: (result, seconds)})."""
    import oracle as O

    def one(i):
        t = time.perf_counter()
        r = O.search(og, [kg.posting(x) for x in qs.central[i]], [kg.posting(x) for x in qs.marginal[i]], qs.k,
                     qs.depth, want_matrices=False, want_candidates=False)
        return i, r, time.perf_counter() - t

    t0 = time.perf_counter()
    if threads <= 1:
        out = [one(i) for i in idx]
    else:
        from concurrent.futures import ThreadPoolExecutor
        with ThreadPoolExecutor(threads) as ex:
            out = list(ex.map(one, idx))
    return time.perf_counter() - t0, {i: (r, dt) for i, r, dt in out}


def _pct(xs, p):
    xs = sorted(xs)
    return xs[min(len(xs) - 1, int(p * len(xs)))] if xs else None


def same_result(gpu, orc):
    """Element-wise identity of one query's answer (north star bar): every RPG's central node,
    S^c, S^m, S^r (exact), PTC flag, node / edge / V_C sets and distance vectors, plus the
    run statistics (terminating levels, relaxation counts)."""
    if len(gpu.rpgs) != len(orc.rpgs):
        return False
    for a, b in zip(gpu.rpgs, orc.rpgs):
        if (a.central_node, a.sc, a.sm, a.score, int(a.ptc)) != (b.central_node, b.sc, b.sm, b.score, int(b.ptc)):
            return False
        for f in ("nodes", "edge_ids", "vc", "cdist", "mdist"):
            if getattr(a, f).tolist() != getattr(b, f).tolist():
                return False
    st = gpu.stats
    return (st["L_central"], st["L_marginal"], st["relax_central"], st["relax_marginal"]) == \
        (orc.Lc, orc.Lm, orc.relax_c, orc.relax_m)


def step_size(cfg, spec, arg):
    if arg:
        return arg
    return 1000 if cfg == 5 else spec.n_queries


def query_set(kg, cfg, spec, rank, world):
    """The config's query set; under weak scaling every rank draws its own set of the same shape."""
    import synth
    if world == 1 or rank == 0:
        return synth.config_queries(kg, cfg)
    if cfg == 5:
        return synth.c5_queries(kg, spec.n_queries, 2005 + 7919 * rank)
    return synth.make_queries(kg, spec.n_queries, spec.n_central, spec.n_marginal, spec.k, spec.depth,
                              2000 + cfg + 7919 * rank)


def chunk(qs, per, i):
    """Step i's queries: chunk i mod (n / per) of the query set."""
    n = len(qs.central)
    nch = max(1, n // per)
    c = i % nch
    return list(range(c * per, min(n, (c + 1) * per)))


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import synth
    spec = synth.CONFIGS[args.config]
    kg = synth.make_kg(args.config)
    qs = synth.config_queries(kg, args.config)
    per = step_size(args.config, spec, args.queries)
    cores = host_cores()
    # each step: a bounded sample of the step's chunk (one query per thread; the oracle takes
    # 5-40 s per config-5 query, so a step is about its slowest query)
    nref = args.ref_queries or min(cores, 8 if args.config >= 4 else 2 * cores)
    og = oracle_graph(kg)

    def idx(s):
        q = chunk(qs, per, s)
        return q[:nref]

    for s in range(args.warmup):
        oracle_run(kg, og, qs, idx(s), cores)
    times, lat = [], []
    for s in range(args.steps):
        dt, res = oracle_run(kg, og, qs, idx(args.warmup + s), cores)
        times.append(dt)
        lat += [t for _, t in res.values()]
    tot = sum(times)
    v = nref * args.steps / tot
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": {"workload": _workload_name(args.config, spec, per), "queries_per_step": nref},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu": cpu_model(),
                             "sample": f"each step: the first {nref} queries of that step's {per}-query chunk of the "
                                       f"config-{args.config} set, oracle/riki_oracle.c as it stands, one query per "
                                       f"thread on {cores} host cores",
                             "query_seconds_p50": _pct(lat, 0.5), "query_seconds_p99": _pct(lat, 0.99)},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="riki", choices=["riki", "reference"])
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--queries", type=int, default=0,
                    help="queries per step (default: config 5 -> 1000-query chunks of its 10k set, else the set)")
    ap.add_argument("--cpu-sample", type=int, default=0,
                    help="oracle queries run one per host thread for cpu_baseline (default 2 per core)")
    ap.add_argument("--cpu-latency", type=int, default=0,
                    help="oracle queries run on one core for its p50/p99 latency (default 6 at C4/C5, else 16)")
    ap.add_argument("--ref-queries", type=int, default=0,
                    help="oracle queries per step for --impl reference (0 = 8 at C4/C5, else 2 per core)")
    ap.add_argument("--latency-queries", type=int, default=40)
    ap.add_argument("--no-cpu", action="store_true", help="skip the oracle (cpu_baseline and the parity gate)")
    ap.add_argument("--no-profile", action="store_true", help="skip the profiling pass (roofline)")
    ap.add_argument("--quick", action="store_true", help="timed region only (for ncu launch lists)")
    ap.add_argument("--slots", type=int, default=0, help="queries in flight per launch (0 = whole step)")
    ap.add_argument("--pull", action="store_true", help="enable the direction-optimising (pull) expansion")
    ap.add_argument("--joint", type=int, default=0, help="1 = joint multi-query traversal for the batch")
    ap.add_argument("--vp", action="store_true",
                    help="vertex-partitioned mode (SURVEY §8(e)): every rank runs the SAME chunks, each pulling "
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
    per = step_size(args.config, spec, args.queries)
    qs = query_set(kg, args.config, spec, 0 if args.vp else rank, 1 if args.vp else world)
    per = min(per, len(qs.central))
    g = P.Graph(kg.n_nodes, kg.src, kg.dst, kg.label_class, kg.term_ptr, kg.postings, device=dev)
    g.set_label_weights(0.5, kg.avg_hops)
    g.set_batch_slots(args.slots or min(per, 1024))
    g.set_direction(1 if args.pull else 0)
    g.set_joint(bool(args.joint))
    if args.vp:
        if dist:
            from paper_2001_06770_b200.dist import init_vertex_partitioned
            init_vertex_partitioned(g)
        else:
            g.dist_init(1, 0, P.riki.dist_unique_id(), mode=1)
    units = 1 if args.vp else world  # VP: all ranks cooperate on the same queries

    # every chunk's query arrays resident in HBM before the timed region
    nchunks = max(1, len(qs.central) // per)
    host_chunks, dev_chunks = [], []
    for c in range(nchunks):
        ids = chunk(qs, per, c)
        cs, ms = [qs.central[i] for i in ids], [qs.marginal[i] for i in ids]
        cp, ct = P.Graph._csr(cs)
        mp, mt = P.Graph._csr(ms)
        host_chunks.append((ids, cs, ms, (cp, ct, mp, mt)))
        dev_chunks.append([torch.from_numpy(x.view(np.int64) if x.dtype == np.uint64 else x.view(np.int32))
                           .to(f"cuda:{dev}") for x in (cp, ct, mp, mt)])
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{dev}")  # > 126 MB L2

    def step_device(i):
        d = dev_chunks[i % nchunks]
        n = len(host_chunks[i % nchunks][0])
        g.search_batch_device(n, d[0].data_ptr(), d[1].data_ptr(), d[2].data_ptr(), d[3].data_ptr(), qs.k, qs.depth)
        return n

    def barrier():
        if dist:
            dist.barrier()

    rdev = f"cuda:{dev}" if not dist or dist.get_backend() == "nccl" else None

    def timed_pass(fn, clocks=None):
        """K steps, each bracketed by CUDA events on the current stream after an L2 flush that
        has completed (the library runs on its own stream); returns per-step ms and queries."""
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        nq = 0
        barrier()
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            torch.cuda.synchronize()
            ev[i][0].record()
            nq += fn(i)
            ev[i][1].record()
        torch.cuda.synchronize()
        barrier()
        return [a.elapsed_time(b) for a, b in ev], nq

    for i in range(args.warmup):
        step_device(args.steps + i)  # chunks not timed first (the timed pass starts at chunk 0)
    torch.cuda.synchronize()
    gc.collect()   # no Python GC pauses inside timed regions
    gc.disable()
    # ---------------- timed region: production path (CUDA-graph level loops, no profiling syncs)
    g.set_profiling(False)
    g.reset_stats()
    with Clocks(dev) as clk:
        step_ms, nq_timed = timed_pass(step_device)
    st_prod = g.stats()
    tot_ms = max_over_ranks(sum(step_ms), device=rdev)  # time = slowest rank
    value = nq_timed * units / (tot_ms / 1000.0)
    if args.quick:
        if rank == 0:
            print(json.dumps({"metric": METRIC, "value": value, "unit": UNIT, "ms_per_step": tot_ms / args.steps,
                              "quick": True, "stats": st_prod}), flush=True)
        return

    # ---------------- profiling pass (same chunks): CUDA events around every expansion launch
    prof = None
    if not args.no_profile:
        g.reset_stats()
        g.set_profiling(True)
        prof_ms, _ = timed_pass(step_device)
        g.set_profiling(False)
        prof = g.stats()
        prof["step_ms"] = prof_ms

    # ---------------- e2e through the host C-ABI (H2D of queries, D2H of results inside)
    res_by_chunk = {}

    def step_e2e(i):
        ids, cs, ms, arrs = host_chunks[i % nchunks]
        rr = g.search_batch(cs, ms, qs.k, qs.depth)  # H2D of the queries, D2H + export of every result
        if dist and not args.vp:  # replicated mode: every shard's results gathered to rank 0
            gather_results(rr, device=rdev)
        if i < nchunks:
            res_by_chunk[i % nchunks] = rr
        return len(ids)

    e2e_step_ms, nq_e2e = timed_pass(step_e2e)
    # bytes moved per step (counted after the timed region from the tensors copied)
    h2d = sum(a.nbytes for a in host_chunks[0][3])
    rr0 = res_by_chunk[0]
    d2h = int(rr0.hdr.nbytes + rr0.score.nbytes + rr0.nodes.nbytes + rr0.edges.nbytes + rr0.vc.nbytes +
              rr0.cd.nbytes + rr0.md.nbytes + rr0.stats.nbytes + rr0.cnt.nbytes) if hasattr(rr0, "hdr") else 0
    e2e_ms = max_over_ranks(sum(e2e_step_ms), device=rdev)
    e2e_value = nq_e2e * units / (e2e_ms / 1000.0)

    # ---------------- single-query latency (one query in flight, host API incl. D2H)
    gc.collect()
    # warm-up: the timed queries run once untimed -- one-time costs (the level-loop CUDA graphs of
    # each H row-width shape, capacity growth of the single-slot workspace) are not query latency
    nlat = min(args.latency_queries, len(qs.central))
    for i in range(nlat):
        g.search(qs.central[i], qs.marginal[i], qs.k, qs.depth)
    lat = []
    for i in range(nlat):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.search(qs.central[i], qs.marginal[i], qs.k, qs.depth)
        b.record()
        torch.cuda.synchronize()
        lat.append(a.elapsed_time(b))
    gc.enable()

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    # relaxations (GTEPS numerator) and levels of the timed chunks
    relax = levels_bits = 0
    V = kg.n_nodes
    for i in range(args.steps):
        c = i % nchunks
        rr = res_by_chunk.get(c)
        if rr is None:
            continue
        for r, cc, mm in zip(rr, host_chunks[c][1], host_chunks[c][2]):
            relax += r.stats["relax_central"] + r.stats["relax_marginal"]
            # frontier bitmap term of §8(d): V*T/8 bytes per query-level of each run (a run
            # ending at L_end expanded levels 0 .. L_end-1)
            levels_bits += max(r.stats["L_central"], 0) * len(cc) + max(r.stats["L_marginal"], 0) * len(mm)
    peak, peak_src = _peaks()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": tot_ms / args.steps, "higher_is_better": True, "scaling": "strong" if args.vp else "weak",
        "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": _workload_name(args.config, spec, per), "queries_per_step_per_gpu": per,
                   "chunks": f"step i runs chunk i mod {nchunks} of the rank's {len(qs.central)}-query set",
                   "l2": "flushed between steps (256 MiB write)",
                   "parallelism": f"vertex-partitioned x{world} (NCCL bit-plane all-gather per level)" if args.vp
                   else f"query-sharded replicas x{world}",
                   "path": "production (CUDA-graph level loops); roofline from a separate profiling pass",
                   "graph_seed": 1000 + synth.GRAPH_OF.get(args.config, args.config),
                   "query_seed": 2000 + args.config},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "results_gathered_to_rank0": bool(dist) and not args.vp},
        "latency_ms": {"p50": _pct(lat, 0.5), "p99": _pct(lat, 0.99), "n": len(lat), "max": max(lat) if lat else None},
        "gteps": relax / (tot_ms / 1000.0) / 1e9 * units if tot_ms else None,
        "relaxations_per_step": relax / args.steps,
        "step_ms": [round(x, 3) for x in step_ms],
        "clocks": clk.summary(),
    }
    if prof is not None:
        # SURVEY §8(d) algorithmic bytes of the expansion (the dominant kernel): 5 B per distinct
        # (edge, level) read + 8 B per distinct (node, level) row header + 1 B per new H cell +
        # the frontier-bitmap term V*T/8 per query-level
        b_edges, b_items, b_cells = 5 * prof["exp_edges"], 8 * prof["exp_items_work"], prof["exp_new_cells"]
        b_bitmap = V * levels_bits // 8
        b_alg = b_edges + b_items + b_cells + b_bitmap
        nl = max(1, prof["expand_launches"])
        exp_s = prof["expand_ms"] / 1e3
        achieved = b_alg / 1e9 / exp_s if exp_s > 0 else 0.0
        traffic, traffic_src = None, None
        try:  # ncu DRAM bytes of the expansion launches of this config (profiles/, committed)
            import glob
            tf = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_expand_traffic_c{args.config}.json")))[-1]
            tj = json.load(open(tf))
            traffic = tj["dram_bytes_per_launch"]
            traffic_src = f"{os.path.relpath(tf, ROOT)}: {tj['dram_bytes_step'] / 1e9:.2f} GB DRAM per step " \
                          f"({tj.get('note', 'ncu')})"
        except Exception:
            pass
        prof_tot = sum(prof["step_ms"])
        qbytes = b_alg / max(1, nq_timed)
        line["roofline"] = {
            "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak if peak else None,
            "traffic": traffic, "traffic_source": traffic_src,
            "kernel": "k_expand + k_expand_heavy (Alg. 1 expansion); CUDA events on the library stream around every "
                      "expansion launch in a profiling pass over the same chunks",
            "achieved_bytes_per_launch": b_alg / nl, "launches_per_step": nl / args.steps,
            "bytes_model": "SURVEY §8(d): 5*P_e + 8*#(f,L) + new cells + V*T/8 per query-level",
            "bytes_per_step": {"edges_5Pe": b_edges / args.steps, "row_headers_8fL": b_items / args.steps,
                               "new_cells": b_cells / args.steps, "bitmap_VT8": b_bitmap / args.steps},
            "builder_model_bytes_per_step": prof["expand_bytes"] / args.steps,
            "builder_model_achieved": prof["expand_bytes"] / 1e9 / exp_s if exp_s > 0 else None,
            "expand_ms_per_step": prof["expand_ms"] / args.steps,
            "expand_share_of_step": prof["expand_ms"] / prof_tot if prof_tot else None,
            "profiling_pass_ms_per_step": prof_tot / args.steps,
            "sections_ms_per_step": {k: x / args.steps for k, x in zip(
                ("central_run", "cg_recovery", "marginal_run", "finalize"), prof["section_ms"])},
            "levels_per_step": prof["levels"] / args.steps,
            "qps_roofline_expansion_bytes": peak * 1e9 / qbytes * units if qbytes else None,
            "qps_frac_of_roofline": value / (peak * 1e9 / qbytes * units) if qbytes else None,
            "peak_source": peak_src}
        # The expansion is bound by RANDOM row accesses, not by streaming bandwidth: every due edge
        # reads its neighbour's H row at a random address and a productive one follows it with a
        # dependent atomicAnd.  Ceiling for that mix, measured on this pool's B200s by
        # tools/randbench.cu (uniformly random 4-byte accesses over 8 GiB; a miss fetches a full
        # 128-byte line): T = (loads - atomics) / load rate + atomics / (load+atomic pair rate).
        try:
            rb = [json.loads(x) for x in open(os.path.join(ROOT, "profiles", "r02_randbench_b200.jsonl"))
                  if x.startswith("{") and '"working_set_mib": 8192' in x]
            r_load = next(x for x in rb if x["pattern"] in ("load", "load.cg"))["g_accesses_per_s"] * 1e9
            r_pair = next(x for x in rb if x["pattern"] in ("load+atomicAnd", "load.cg+atomicAnd"))["g_accesses_per_s"] * 1e9 / 2
            loads, atoms = prof["exp_edges"], prof.get("exp_atomics", 0)
            t_ceil = (loads - atoms) / r_load + atoms / r_pair
            line["random_access_roofline"] = {
                "bound": "random 128-byte line fetches (HBM latency/concurrency), measured",
                "load_rate_g_per_s": r_load / 1e9, "pair_rate_g_per_s": r_pair / 1e9,
                "source": "profiles/r02_randbench_b200.jsonl (tools/randbench.cu, 8 GiB working set)",
                "h_row_loads_per_step": loads / args.steps, "atomics_per_step": atoms / args.steps,
                "ceiling_ms_per_step": t_ceil * 1e3 / args.steps, "expand_ms_per_step": exp_s * 1e3 / args.steps,
                "frac": t_ceil / exp_s if exp_s > 0 else None,
                "note": "frac > 1 is possible: hub rows hit in L2, the uniform-random ceiling assumes none do"}
        except Exception as e:  # noqa: BLE001 -- reported, never fatal
            line["random_access_roofline"] = {"error": str(e)}
        line["gpu_launches"] = int(prof["kernel_launches"])
        line["gpu_launches_note"] = "kernels launched for the timed steps' work, counted in the profiling pass " \
                                    "(the production pass replays the same kernels from CUDA graphs)"
    else:
        line["gpu_launches"] = int(st_prod["kernel_launches"])
    if args.vp:
        di = g.dist_info()
        line["vp"] = {"nranks": di["nranks"], "bounds": di["bounds"].tolist(), "exchanges": di["exchanges"],
                      "exchanged_bytes": di["exchanged_bytes"]}
    if world == 1 and not args.no_cpu and 0 in res_by_chunk:
        # ---------------- the oracle on a bounded sample of chunk 0: latency on one core, then
        # throughput one query per host core; its answers gate this line (parity)
        cores = host_cores()
        big = args.config >= 4
        n1 = args.cpu_latency or (6 if big else 16)
        n = args.cpu_sample or 2 * cores
        ids0 = host_chunks[0][0]
        n1 = min(n1, len(ids0))
        n = min(n, len(ids0) - n1)
        og = oracle_graph(kg)
        dt1, r1 = oracle_run(kg, og, qs, ids0[:n1], 1)
        dt, rn = oracle_run(kg, og, qs, ids0[n1:n1 + n], cores)
        lat1 = [t for _, t in r1.values()]
        tc = sum(r.extra["t_central"] for r, _ in r1.values())
        tm = sum(r.extra["t_marginal"] for r, _ in r1.values())
        line["cpu_baseline"] = {
            "value": n / dt if n else None, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu": cpu_model(),
            "sample": f"queries {n1}..{n1 + n - 1} of chunk 0 ({per} queries) of the same set, one query per thread "
                      f"on {cores} host cores (oracle/riki_oracle.c as it stands)",
            "single_core": {"value": n1 / dt1 if n1 else None, "cores": 1,
                            "latency_s_p50": _pct(lat1, 0.5), "latency_s_p99": _pct(lat1, 0.99),
                            "phase_split": {"central_run_and_cg_recovery_s": tc / max(1, n1),
                                            "marginal_run_attach_rpg_s": tm / max(1, n1)},
                            "sample": f"queries 0..{n1 - 1} of chunk 0, one at a time"}}
        rr0 = res_by_chunk[0]
        checked = identical = 0
        bad = []
        for j, (r, _) in list(r1.items()) + list(rn.items()):
            pos = ids0.index(j)
            checked += 1
            if same_result(rr0[pos], r):
                identical += 1
            else:
                bad.append(j)
        line["parity"] = {"checked": checked, "identical": identical, "mismatched_queries": bad[:16],
                          "compared": "every RPG (central node, S^c, S^m, S^r exact, PTC, node/edge/V_C sets, "
                                      "distances) and per-run terminating levels and relaxation counts, GPU "
                                      "(e2e pass, chunk 0) vs oracle",
                          "oracle_activations": "the oracle's own fine weights + coarsening"}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
