#!/bin/bash
# Run on the GPU box:  tools/profile_kernel.sh <tag> <kernel-regex>
# Full ncu capture (--set full, source) of the LONGEST launch matching <kernel-regex> in one
# quick bench step (warmup 1, steps 1), picked from a duration pass over the same run.
set -e
T=$1; K=$2
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$K" --csv \
    --log-file gpurun_out/${T}_dur.csv python bench.py --steps 1 --warmup 1 --quick > gpurun_out/${T}_dur.log 2>&1
SKIP=$(python - "$T" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(f"gpurun_out/{sys.argv[1]}_dur.csv")) if len(r) > 10]
hdr, rows = rows[0], rows[1:]
ix = {h: i for i, h in enumerate(hdr)}
d = [float(r[ix["Metric Value"]]) for r in rows]
print(max(range(len(d)), key=lambda i: d[i]))
PY
)
echo "capture ordinal $SKIP"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s $SKIP -c 1 \
    -o gpurun_out/${T}_full python bench.py --steps 1 --warmup 1 --quick > gpurun_out/${T}_full.log 2>&1
echo done
