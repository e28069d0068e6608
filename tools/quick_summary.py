import json, sys
for ln in open(sys.argv[1]):
    ln = ln.strip()
    i = ln.find('{"metric"')
    if i < 0:
        continue
    try:
        d = json.loads(ln[i:])
    except Exception:
        continue
    st = d.get("stats")
    if not st:
        continue
    n = max(1, st["queries"] // 200)
    print(round(d["value"]), "q/s", round(d["ms_per_step"], 2), "ms  expand", round(st["expand_ms"] / n, 2),
          "sections", [round(x / n, 2) for x in st["section_ms"]], "levels", st["levels"] / n)
