"""Summarise tools/profile_round.sh output into profiles/<R>_*.  usage: profile_summary.py r01"""
import csv, collections, json, os, subprocess, sys
R = sys.argv[1]
G = "gpurun_out"
os.makedirs("profiles", exist_ok=True)

def rows(path):
    hdr, out = None, []
    for r in csv.reader(open(path)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            out.append(dict(zip(hdr, r)))
    return out

# ---- launch list: the last (timed) step starts after the last torch fill (L2 flush)
lst = rows(f"{G}/{R}_launches.csv")
fills = [i for i, d in enumerate(lst) if "at::" in d["Kernel Name"] and "fill" in d["Kernel Name"].lower()]
step = lst[fills[-1] + 1:]
agg = collections.defaultdict(lambda: [0, 0.0])
for d in step:
    n = d["Kernel Name"].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
    agg[n][0] += 1
    agg[n][1] += float(d["Metric Value"]) / 1e3
tot = sum(v[1] for v in agg.values())
with open(f"profiles/{R}_launch_list_summary.txt", "w") as f:
    f.write(f"# one bench step (config 2, 200 queries): {len(step)} launches, sum of device times {tot/1e3:.3f} ms\n")
    f.write("# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised launches)\n")
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        f.write(f"{t:10.1f} us {100*t/tot:5.1f}% {c:4d}  {n}\n")
# ---- expansion DRAM traffic per launch (timed step only: second half of the expansion launches)
ex = rows(f"{G}/{R}_expand_dram.csv")
by = collections.defaultdict(dict)
for d in ex:
    by[d["ID"]][d["Metric Name"]] = float(d["Metric Value"])
    by[d["ID"]]["name"] = d["Kernel Name"]
ids = sorted(by, key=int)
n_last = sum(c for n, (c, t) in agg.items() if n.startswith("k_expand"))  # expansion launches per step
half = ids[-n_last:]
dram = sum(by[i]["dram__bytes_read.sum"] + by[i]["dram__bytes_write.sum"] for i in half)
l2 = sum(by[i].get("lts__t_bytes.sum", 0) for i in half)
t_ns = sum(by[i]["gpu__time_duration.sum"] for i in half)
alg = None
try:
    b = json.loads(open(f"{G}/{R}_list.log").read().strip().splitlines()[-1])
    alg = b["stats"]["expand_bytes"] / max(1, b["stats"]["queries"] // 200)
except Exception:
    pass
out = {"round": R, "launches": len(half), "algorithmic_bytes_step": alg, "dram_bytes_step": dram, "dram_bytes_per_launch": dram / max(1, len(half)),
       "l2_bytes_step": l2, "device_ms_step": t_ns / 1e6,
       "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:k_expand (timed step)"}
json.dump(out, open(f"profiles/{R}_expand_traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
# ---- full capture of the largest launch
rep = f"{G}/{R}_expand_full.ncu-rep"
if os.path.exists(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    hdr, units, d = rr[0], rr[1], rr[2]
    keys = ["Grid Size", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
            "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__average_warp_latency_per_inst_issued.ratio",
            "launch__registers_per_thread", "sm__inst_executed.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
            "l1tex__t_requests_pipe_lsu_mem_global_op_atom.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
            "lts__t_sectors_op_read.sum", "lts__t_sectors_op_atom.sum", "lts__t_sectors_op_red.sum", "lts__t_sectors_op_write.sum",
            "smsp__inst_executed.sum", "smsp__sass_inst_executed_op_global_atom.sum"]
    with open(f"profiles/{R}_expand_full_summary.txt", "w") as f:
        f.write("# ncu --set full --clock-control none -k regex:k_expand -s <ordinal> -c 1: the longest k_expand launch of the run (marginal flood level), picked from the DRAM pass\n")
        for k in keys:
            if k in hdr:
                f.write(f"{k} = {d[hdr.index(k)]} {units[hdr.index(k)]}\n")
        st = sorted([(h, d[i]) for i, h in enumerate(hdr) if "smsp__average_warps_issue_stalled" in h
                     and h.endswith("per_issue_active.ratio")], key=lambda x: -float(x[1] or 0))[:8]
        f.write("# top stall reasons (cycles per issued instruction)\n")
        for h, v in st:
            f.write(f"{h} = {v}\n")
    print(open(f"profiles/{R}_expand_full_summary.txt").read())
