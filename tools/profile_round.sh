#!/bin/bash
# Run on the GPU box:  tools/profile_round.sh r01
# 1) launch list of one bench step (device time of every launch, cold-cache, serialised)
# 2) DRAM bytes of every expansion launch of one step (the bench's "traffic")
# 3) ncu --set full of the longest k_expand launch (marginal flood level), picked from 2)
set -e
R=${1:-r01}
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/${R}_launches.csv python bench.py --steps 1 --warmup 1 --quick > gpurun_out/${R}_list.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
    --clock-control none -k regex:k_expand --csv --log-file gpurun_out/${R}_expand_dram.csv \
    python bench.py --steps 1 --warmup 1 --quick > gpurun_out/${R}_dram.log 2>&1
# ordinal (among the regex:k_expand launches above) of the longest k_expand launch of the run
SKIP=$(python - "$R" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(f"gpurun_out/{sys.argv[1]}_expand_dram.csv")) if len(r) > 10]
hdr, rows = rows[0], rows[1:]
ix = {h: i for i, h in enumerate(hdr)}
ids, dur, name = [], {}, {}
for r in rows:
    i = int(r[ix["ID"]])
    if i not in name:
        ids.append(i)
        name[i] = r[ix["Kernel Name"]]
    if r[ix["Metric Name"]] == "gpu__time_duration.sum":
        dur[i] = float(r[ix["Metric Value"]])
best = max((i for i in ids if "k_expand_heavy" not in name[i]), key=lambda i: dur.get(i, 0))
print(ids.index(best))
PY
)
echo "full capture: k_expand launch ordinal $SKIP"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_expand -s $SKIP -c 1 \
    -o gpurun_out/${R}_expand_full python bench.py --steps 1 --warmup 1 --quick > gpurun_out/${R}_full.log 2>&1
echo profile_done
# 4) DRAM bytes and duration of EVERY launch of one step: per-kernel achieved DRAM GB/s
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 \
    --csv --log-file gpurun_out/${R}_all_dram.csv python bench.py --steps 1 --warmup 1 --quick > gpurun_out/${R}_all_dram.log 2>&1
echo dram_done
