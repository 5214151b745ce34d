# round 2, call v: block renumberings (bx x by quads per seed tile) at 4 KB first-pass scratch; 5-CTA build
O=gpurun_out/r02v
mkdir -p $O
sw() { timeout 600 python tools/sweep_ts.py "$@" 2>&1 | grep -E '"ts"|lt plan\] (tiles|dataflow)' | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('[lt plan]'): print('   ', l.strip()); continue
    d=json.loads(l); print('$LT_LIB_TAG', ' '.join(sys.argv[1:]), '|', d.get('ts'), d.get('ms_per_step'), '%.4g'%d.get('value',0), d.get('wide'), d.get('smem'), d.get('colors'), d.get('error',''))" "$@"; }
export LT_DEBUG_PLAN=1
for v in base n5; do
  if [ "$v" = base ]; then unset LT_LIB_PATH; else export LT_LIB_PATH=$PWD/paper_1708_03183_b200/libltcuda_$v.so; fi
  export LT_LIB_TAG=$v
  sw 4 4096 2048 --ts 16 --steps 3 --renumber morton
  sw 4 4096 2048 --ts 12 --steps 3 --renumber block:3x2
  sw 4 4096 2048 --ts 12 --steps 3 --renumber block:2x3
  sw 4 4096 2048 --ts 18 --steps 3 --renumber block:3x3
  sw 4 4096 2048 --ts 16 --steps 3 --renumber block:4x2
  sw 4 4096 2048 --ts 20 --steps 3 --renumber block:5x2
  sw 4 4096 2048 --ts 24 --steps 3 --renumber block:4x3
  sw 3 --ts 32 --steps 3 --renumber morton
  sw 3 --ts 24 --steps 3 --renumber block:4x3
  sw 3 --ts 32 --steps 3 --renumber block:4x4
  sw 3 --ts 40 --steps 3 --renumber block:5x4
  sw 3 --ts 36 --steps 3 --renumber block:6x3
  sw 3 --ts 48 --steps 3 --renumber block:6x4
done > $O/sweep.txt 2>&1
unset LT_LIB_PATH
timeout 300 python tools/sweep_ts.py 2 --chains 10 --ts 32 --steps 10 2>&1 | grep '"ts"' >> $O/sweep.txt
grep -v "^    \[lt plan\] tiles" $O/sweep.txt
