"""Expansion DRAM traffic of one bench step from an ncu per-launch DRAM capture
(tools/profile_r02.sh ..._all_dram.csv) -> profiles/<tag>_expand_traffic_c<cfg>.json, the file
bench.py reads for roofline.traffic; also a per-kernel summary text.
usage: traffic_json.py <all_dram.csv> <tag> <cfg> <queries per step>"""
import collections
import csv
import json
import sys

src, tag, cfg, nq = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
rows = [r for r in csv.reader(open(src)) if len(r) > 10]
hdr, rows = rows[0], rows[1:]
ix = {h: i for i, h in enumerate(hdr)}
per, name, order = collections.defaultdict(dict), {}, []
for r in rows:
    i = int(r[ix["ID"]])
    if i not in name:
        name[i] = r[ix["Kernel Name"]]
        order.append(i)
    per[i][r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
fills = [i for i in order if "fill" in name[i].lower() and "at::" in name[i]]
step = [i for i in order if i > fills[-1]]  # the timed step follows the last L2-flush fill
exp = [i for i in step if "k_expand" in name[i]]
dram = lambda i: per[i].get("dram__bytes_read.sum", 0) + per[i].get("dram__bytes_write.sum", 0)
tot_b = sum(dram(i) for i in exp)
tot_t = sum(per[i].get("gpu__time_duration.sum", 0) for i in exp)
step_t = sum(per[i].get("gpu__time_duration.sum", 0) for i in step)
out = {"config": cfg, "queries_per_step": nq, "launches": len(exp), "dram_bytes_step": tot_b,
       "dram_bytes_per_launch": tot_b / max(1, len(exp)), "expand_ns_step": tot_t,
       "expand_share_of_step_ncu": tot_t / step_t if step_t else None,
       "dram_gbs_expand": tot_b / tot_t if tot_t else None,
       "note": f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
               f"--clock-control none, one step of bench.py --config {cfg} (plain launches), source {src}"}
json.dump(out, open(f"profiles/{tag}_expand_traffic_c{cfg}.json", "w"), indent=1)
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for i in step:
    n = name[i].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
    a = agg[n]
    a[0] += 1
    a[1] += per[i].get("gpu__time_duration.sum", 0)
    a[2] += dram(i)
with open(f"profiles/{tag}_kernels_c{cfg}.txt", "w") as f:
    f.write(f"# one bench step of config {cfg} ({nq} queries): {len(step)} launches, {step_t / 1e6:.2f} ms summed "
            f"device time (ncu, cold-cache, serialised launches; --clock-control none)\n")
    f.write("# ms  share  launches  DRAM GB  DRAM GB/s  kernel\n")
    for n, (c, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        f.write(f"{t / 1e6:9.2f} {100 * t / step_t:5.1f}% {c:6d} {b / 1e9:9.2f} {b / t if t else 0:8.0f}  {n}\n")
print(json.dumps(out))
