#!/bin/bash
# Run on the GPU box: tools/ab_variants.sh <tag> <config> <steps> lib1 lib2 ...
# quick bench (production path, timed region only) of each library variant, one process each;
# extra bench arguments in $AB_ARGS
T=$1; C=$2; S=$3; shift 3
for L in "$@"; do
  echo "== $L" >> gpurun_out/${T}_ab_c${C}.log
  RIKI_LIB=$PWD/paper_2001_06770_b200/$L python bench.py --config $C --steps $S --warmup 2 --quick --no-cpu $AB_ARGS >> gpurun_out/${T}_ab_c${C}.log 2>&1
done
