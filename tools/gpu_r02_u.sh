# round 2, call u: smaller first-pass record scratch (shortest chunk) -> more CTAs per SM?
O=gpurun_out/r02u
mkdir -p $O
sw() { timeout 600 python tools/sweep_ts.py "$@" 2>&1 | grep -E '"ts"|lt plan\] (tiles|dataflow)' | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('[lt plan]'): print('   ', l.strip()); continue
    d=json.loads(l); print('$LT_LIB_TAG s1=$LT_SCRATCH1_KB', sys.argv[1:], d.get('ts'), d.get('ms_per_step'), '%.4g'%d.get('value',0), d.get('wide'), d.get('smem'), d.get('error',''))" "$@"; }
export LT_DEBUG_PLAN=1
for v in base n5; do
  if [ "$v" = base ]; then unset LT_LIB_PATH; else export LT_LIB_PATH=$PWD/paper_1708_03183_b200/libltcuda_$v.so; fi
  export LT_LIB_TAG=$v
  for s1 in 8 4 2 1; do
    export LT_SCRATCH1_KB=$s1
    sw 4 4096 2048 --ts 16 --steps 3
    sw 3 --ts 16,32 --steps 3
  done
done > $O/sweep.txt 2>&1
cat $O/sweep.txt
