#!/bin/bash
# usage: make -C paper_1708_03183_b200/csrc variant NAME=x DEFS="-DKNOB=v"; bash tools/gpu_ab.sh base x
# A/B: bench configs 2 and 3 with each library variant given as argument (default lib = "base")
summ() { python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('  c%s value %.4g ms %.4f frac %.4f clk %s' % (d['config']['p']+1, d['value'], d['ms_per_step'], d['roofline']['frac'], d['clocks']['sm_mhz']))"; }
for v in "$@"; do
  if [ "$v" = base ]; then unset LT_LIB_PATH; else export LT_LIB_PATH=$PWD/paper_1708_03183_b200/libltcuda_$v.so; fi
  echo "== $v"
  for c in 2 3; do python bench.py --config $c --steps 5 --no-cpu-baseline --no-e2e $BENCH_ARGS 2>/dev/null | summ; done
done
