#!/bin/bash
# usage: bash tools/ab_variants.sh "base v1 v2" "<sweep args>" ...   (GPU box)
# Each library variant (libltcuda_<v>.so; "base" = libltcuda.so) runs tools/sweep_ts.py
# with each argument set, twice in alternating order; one summary line per run.
VARS=$1; shift
for rep in 1 2; do
  for v in $VARS; do
    if [ "$v" = base ]; then unset LT_LIB_PATH; else export LT_LIB_PATH=$PWD/paper_1708_03183_b200/libltcuda_$v.so; fi
    for a in "$@"; do
      python tools/sweep_ts.py $a 2>&1 | grep '"ts"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v rep$rep [$a]', d.get('ts'), d.get('ms_per_step'), '%.4g'%d.get('value',0), d.get('wide'), d.get('smem'), d.get('error',''))"
    done
  done
done
