#!/bin/bash
# Run on the GPU box:  tools/profile_r02.sh <tag> <config>
# 1) launch list of one bench step of <config> (device time of every launch, cold-cache, serialised)
# 2) DRAM bytes + duration of every launch of that step (per-kernel achieved DRAM GB/s, the
#    expansion's traffic for the bench's roofline.traffic)
# 3) ncu --set full --import-source of the longest k_expand launch (picked from 2)
set -e
T=$1; C=${2:-5}
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
B="python bench.py --config $C --steps 1 --warmup 1 --quick --no-cpu"
# plain launches (kernels inside the CUDA-graph level loops are not listed one by one)
export RIKI_NO_GRAPHS=1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -c 6000 --csv --log-file gpurun_out/${T}_c${C}_all_dram.csv $B > gpurun_out/${T}_c${C}_dram.log 2>&1
echo dram_done
if [ "${FULL:-1}" = "0" ]; then exit 0; fi
SKIP=$(python - "$T" "$C" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(f"gpurun_out/{sys.argv[1]}_c{sys.argv[2]}_all_dram.csv")) if len(r) > 10]
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
exp = [i for i in ids if name[i].startswith("void <unnamed>::k_expand") or "k_expand<" in name[i]]
light = [i for i in exp if "k_expand_heavy" not in name[i]]
best = max(light, key=lambda i: dur.get(i, 0))
print(exp.index(best))
PY
)
echo "full capture: k_expand launch ordinal $SKIP"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_expand -s $SKIP -c 1 \
    -o gpurun_out/${T}_c${C}_expand_full $B > gpurun_out/${T}_c${C}_full.log 2>&1
echo profile_done
