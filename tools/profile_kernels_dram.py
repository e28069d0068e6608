"""Per-kernel DRAM throughput of one bench step from profile_round.sh step 4.
usage: profile_kernels_dram.py r01e   ->  profiles/<R>_kernels_dram.txt"""
import collections
import csv
import json
import sys

R = sys.argv[1]
rows, hdr = [], None
for r in csv.reader(open(f"gpurun_out/{R}_all_dram.csv")):
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        rows.append(dict(zip(hdr, r)))
launch = collections.OrderedDict()
for d in rows:
    k = int(d["ID"])
    e = launch.setdefault(k, {"name": d["Kernel Name"]})
    v = float(d["Metric Value"].replace(",", ""))
    u = d.get("Metric Unit", "")
    if d["Metric Name"] == "gpu__time_duration.sum":
        e["ns"] = v * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(u, 1)
    else:
        e[d["Metric Name"]] = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
ids = list(launch)
fills = [i for i in ids if "at::" in launch[i]["name"] and "fill" in launch[i]["name"].lower()]
step = [launch[i] for i in ids[ids.index(fills[-1]) + 1:]] if fills else [launch[i] for i in ids]
try:
    peak = float(json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"])
except Exception:
    peak = 6650.0
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for e in step:
    n = e["name"].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
    a = agg[n]
    a[0] += 1
    a[1] += e.get("ns", 0.0)
    a[2] += e.get("dram__bytes_read.sum", 0.0) + e.get("dram__bytes_write.sum", 0.0)
tot_ns = sum(a[1] for a in agg.values())
with open(f"profiles/{R}_kernels_dram.txt", "w") as f:
    f.write(f"# one bench step (config 2): per-kernel DRAM bytes / device time (ncu, cold cache, serialised); "
            f"peak {peak:.0f} GB/s\n# kernel  launches  time_us  share  dram_MB  GB/s  frac_of_peak\n")
    for n, (c, ns, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        gbs = b / ns if ns else 0.0
        f.write(f"{n:48s} {c:5d} {ns / 1e3:10.1f} {ns / tot_ns:6.1%} {b / 1e6:10.1f} {gbs:8.1f} {gbs / peak:6.3f}\n")
print(open(f"profiles/{R}_kernels_dram.txt").read())
