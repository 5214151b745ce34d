# round 2, call y: 168-register build where shared memory caps the CTAs per SM at 3 (A/B by LT_NO_WIDE3)
O=gpurun_out/r02y
mkdir -p $O
export LT_LIB_PATH=$PWD/paper_1708_03183_b200/libltcuda_w3.so
for rep in 1 2; do
for off in 1 0; do
  if [ $off = 1 ]; then export LT_NO_WIDE3=1; else unset LT_NO_WIDE3; fi
  for a in "4 4096 2048 --ts 24 --steps 5" "3 --ts 24 --steps 5 --renumber none" "3 --ts 40 --steps 5 --renumber block:4x5"; do
    timeout 600 python tools/sweep_ts.py $a 2>&1 | grep '"ts"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('nowide3=$off rep$rep [$a]', d.get('ts'), d.get('ms_per_step'), '%.4g'%d.get('value',0), d.get('wide'), d.get('smem'), d.get('error',''))"
  done
done
done > $O/ab.txt 2>&1
cat $O/ab.txt
