"""Per-CUDA-source-line instruction and stall totals of one ncu report (cuda,sass view):
usage: ncu_lines.py rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur_file, hdr, agg = None, None, []
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        iI = hdr.index("Instructions Executed")
        iW = hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0] != "":  # a CUDA source line (its totals)
        try:
            agg.append((cur_file, int(r[0]), r[1][:100], int(r[iI] or 0), int(r[iW] or 0)))
        except ValueError:
            pass
ti = sum(a[3] for a in agg) or 1
tw = sum(a[4] for a in agg) or 1
print(f"warp inst {ti/1e6:.1f}M  stall samples {tw}")
for f, ln, src, ins, st in sorted(agg, key=lambda a: -a[3])[:top]:
    print(f"{ins/1e6:8.1f}M {100*ins/ti:5.1f}%  st {100*st/tw:5.1f}%  {f}:{ln:<5d} {src.strip()[:90]}")
