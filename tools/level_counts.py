"""Summarise RIKI_LEVELS=1 stderr ([riki-level] lines) of the LAST search call: per phase and level,
active slots, frontier items, heavy chunks, edges walked and new cells."""
import re
import sys

calls, cur = [], None
for ln in open(sys.argv[1]):
    m = re.match(r"\[riki-level\] ph=(\d) l=(\d+) active=(\d+) items=(\d+) heavy_chunks=(\d+) edges=(\d+) cells=(\d+)", ln)
    if not m:
        continue
    ph, l, act, items, hv, e, c = map(int, m.groups())
    if ph == 0 and l == 0:
        cur = []
        calls.append(cur)
    cur.append((ph, l, act, items, hv, e, c))
last = calls[-1]
print(f"{'ph':>2} {'l':>3} {'active':>6} {'items':>10} {'heavy':>7} {'edges':>11} {'cells':>10}")
for r in last:
    print(f"{r[0]:2d} {r[1]:3d} {r[2]:6d} {r[3]:10d} {r[4]:7d} {r[5]:11d} {r[6]:10d}")
for ph in (0, 1):
    rs = [r for r in last if r[0] == ph]
    print(f"phase {ph}: items {sum(r[3] for r in rs)} edges {sum(r[5] for r in rs)} cells {sum(r[6] for r in rs)}")
