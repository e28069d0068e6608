#!/bin/bash
# usage (on the GPU box): tools/variants.sh name1 name2 ...   (variants/lib_<name>.so)
# Runs the quick bench for each variant, two rounds interleaved, prints q/s and expansion ms/step.
for round in 1 2; do
  for v in "$@"; do
    out=$(RIKI_LIB=variants/lib_${v%%+*}.so timeout 200 python bench.py --steps 5 --warmup 2 --quick $( [[ $v == *+push ]] && echo --push-only ) 2>&1 | tail -1)
    echo "$v $out"
  done
done
