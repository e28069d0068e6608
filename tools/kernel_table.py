"""Per-kernel totals of an ncu --csv launch list: device time, DRAM bytes, L2 hit rate, L2
atomic requests.  usage: kernel_table.py file.csv [file2.csv ...]"""
import collections
import csv
import re
import sys

UNIT = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1, "second": 1e3,
        "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
for fn in sys.argv[1:]:
    hdr, launch = None, collections.OrderedDict()
    for r in csv.reader(open(fn)):
        if "Kernel Name" in r:
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        e = launch.setdefault(int(d["ID"]), {"name": d["Kernel Name"]})
        v = float(d["Metric Value"].replace(",", "") or 0)
        e[d["Metric Name"]] = v * UNIT.get(d.get("Metric Unit", ""), 1)
    agg = collections.OrderedDict()
    for e in launch.values():
        n = re.sub(r"\(.*", "", e["name"]).replace("void <unnamed>::", "")
        a = agg.setdefault(n, collections.Counter())
        a["n"] += 1
        a["ms"] += e.get("gpu__time_duration.sum", 0)
        a["rd"] += e.get("dram__bytes_read.sum", 0)
        a["wr"] += e.get("dram__bytes_write.sum", 0)
        a["hitw"] += e.get("lts__t_sector_hit_rate.pct", 0) * e.get("gpu__time_duration.sum", 0)
        a["atom"] += e.get("lts__t_requests_srcunit_tex_op_atom.sum", 0)
    tot = sum(a["ms"] for a in agg.values())
    print(f"== {fn}: {len(launch)} launches, {tot:.2f} ms")
    for n, a in sorted(agg.items(), key=lambda x: -x[1]["ms"]):
        if a["ms"] < 0.002 * tot:
            continue
        print(f"  {n[:48]:48s} {a['n']:5d} {a['ms']:9.3f} ms {100*a['ms']/tot:5.1f}%  rd {a['rd']/1e9:8.2f} GB  wr {a['wr']/1e9:7.2f} GB"
              f"  {(a['rd']+a['wr'])/max(a['ms'],1e-9)/1e6:6.2f} TB/s  hit {a['hitw']/max(a['ms'],1e-9):5.1f}%  atom {a['atom']/1e6:8.1f} M")
