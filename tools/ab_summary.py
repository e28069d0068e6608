"""Collect the round-2 A/B quick-bench values (gpurun_out/r02*_ab_c*.log) into one text file with
what each variant was (profiles/r02_ab_experiments.txt)."""
import glob
import json
import os
import re

NOTES = {
    "r02f": "libriki.so = bounded RPG recovery + u64 expansion at 6 blocks/SM; vb = u64 at 8 blocks (spills); "
            "vc = EXP_MINB 7 (same 32 registers)",
    "r02f_eager": "RIKI_EAGER_RPG=1: every attached candidate's RPG recovered (round-1 behaviour)",
    "r02g": "after the vertex-partitioned push commit (bounded recovery chosen by candidate-set size)",
    "r02h": "libriki.so = lane's unrolled atomics issued together (EXP_BATCH_ATOM=1) + row-width groups; "
            "vd = one atomic at a time",
    "r02h_nogroups": "RIKI_NO_ROW_GROUPS=1: one sub-batch at the widest row width",
    "r02i_s16": "--slots 16 (queries in flight)", "r02i_s32": "--slots 32", "r02i_s128": "--slots 128 (memory-capped)",
    "r02j": "libriki.so = candidate appends gated by one vote; vd = without; vh4/vh8 = grouped H layout HGRP 4/8",
    "r02j_w1": "RIKI_RPG_WAVES=1 (one flush wave); at C2 also RIKI_BOUNDED_RPG=1",
    "r02k": "run-to-run noise: the same libraries repeated (vd, libriki, vd, libriki, ve)",
    "r02l": "EXP_UNROLL 4 (vu4) and HEAVY_UNROLL 4 (vhu4) against the default, each twice",
    "r02q_nob": "the same library with RIKI_NO_BUCKETS=1 (the default path)",
    "r02q": "destination-bucketed relaxation (on by default for V >= 4M) vs RIKI_NO_BUCKETS=1 (r02q_nob), each twice; C2 unaffected",
    "r02n": "EXP_SMALL 4 (libriki.so: ranges of <= 4 due edges walked lane-locally) vs EXP_SMALL 0 (vs0), each twice",
}
out = ["# Round-2 A/B experiments: quick bench (production path, timed region only; "
       "tools/ab_variants.sh), one process per library variant, values in queries/s.",
       "# Run-to-run noise is about +-3 % (r02k), so differences below that are not significant.", ""]
for f in sorted(glob.glob("gpurun_out/r02*_ab_c*.log")):
    tag, cfg = re.match(r"gpurun_out/(r02\w*?)_ab_c(\d)\.log", f).groups()
    out.append(f"## {tag} config {cfg}: {NOTES.get(tag, '')}")
    lib = None
    for ln in open(f):
        if ln.startswith("== "):
            lib = ln[3:].strip()
        elif ln.startswith("{"):
            try:
                d = json.loads(ln)
                out.append(f"   {lib:24s} {d['value']:10.1f} q/s   {d['ms_per_step']:9.2f} ms/step")
            except Exception:
                pass
    out.append("")
os.makedirs("profiles", exist_ok=True)
open("profiles/r02_ab_experiments.txt", "w").write("\n".join(out) + "\n")
print("\n".join(out))
