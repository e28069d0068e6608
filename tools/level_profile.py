"""Per-level kernel times of the last bench step in an ncu launch list (tools/launches.py CSV)."""
import csv
import io
import re
import sys

txt = open(sys.argv[1]).read()
rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
names = [re.sub(r"^(void )?(<unnamed>::)?", "", r["Kernel Name"].split("(")[0]) for r in rows]
begins = [j for j, n in enumerate(names) if n.startswith("k_phase_begin")]
st = begins[-2]
ph, lvl, line = -1, 0, {}
def flush():
    if line:
        print(f"ph{ph} l{lvl:2d} " + "  ".join(f"{k}={v:7.1f}" for k, v in line.items()))
for j in range(st, len(rows)):
    n, t = names[j], float(rows[j]["Metric Value"]) / 1000
    if n.startswith("k_phase_begin"):
        flush(); line = {}; ph += 1; lvl = 0
        continue
    if n.startswith("k_plan"):
        flush(); line = {}; lvl += 1
    key = n.split("<")[0][2:]
    line[key] = line.get(key, 0) + t
flush()
