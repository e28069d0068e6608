import json, sys, collections
res = collections.defaultdict(list)
for ln in open(sys.argv[1]):
    if " {" not in ln:
        continue
    name, js = ln.split(" ", 1)
    try:
        d = json.loads(js)
    except Exception:
        continue
    res[name].append((d["value"], d["stats"]["expand_ms"] / 5))
for n, v in res.items():
    print(f"{n:10s} q/s {[round(x[0]) for x in v]}  expand ms/step {[round(x[1], 2) for x in v]}")
