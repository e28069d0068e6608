"""Brief of one ncu report: key throughput metrics, top stall reasons, and the SASS lines
carrying the most stall samples (with a few lines of context).  usage: ncu_brief.py rep [nctx]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
nctx = int(sys.argv[2]) if len(sys.argv) > 2 else 4
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
hdr, units, d = rr[0], rr[1], rr[2]
keys = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__average_warp_latency_per_inst_issued.ratio"]
for k in keys:
    if k in hdr:
        print(f"{k} = {d[hdr.index(k)][:90]} {units[hdr.index(k)]}")
st = sorted([(h, d[i]) for i, h in enumerate(hdr) if "smsp__average_warps_issue_stalled" in h
             and h.endswith("per_issue_active.ratio")], key=lambda x: -float(x[1] or 0))[:6]
for h, v in st:
    print(f"  stall {h.split('stalled_')[1].split('_per')[0]:24s} {float(v):7.2f}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
h2 = rows[1]
body = rows[2:]
iS, iW, iI = h2.index("Source"), h2.index("Warp Stall Sampling (All Samples)"), h2.index("Instructions Executed")
tw = sum(int(r[iW]) for r in body) or 1
ti = sum(int(r[iI]) for r in body) or 1
print(f"SASS lines {len(body)}, warp inst {ti}, stall samples {tw}")
shown = set()
for j in sorted(range(len(body)), key=lambda j: -int(body[j][iW]))[:12]:
    if int(body[j][iW]) < tw * 0.01:
        break
    print("-----")
    for k in range(max(0, j - nctx), j + 1):
        r = body[k]
        print(f"{k:5d} {int(r[iI])/1e6:7.2f}M {100*int(r[iW])/tw:5.1f}%  {r[iS].strip()[:90]}")
