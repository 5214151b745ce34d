# round 2, call n: grouped items v2 (apply RA rows, minv/axpy per field) at larger tiles / fewer CTAs;
# controls: nogroup (same source, LT_GROUPED=0), b4 (commit b4d8c57, before the TMA code)
O=gpurun_out/r02n
mkdir -p $O
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,power.limit,clocks_event_reasons.active --format=csv > $O/smi.txt
for v in base nogroup b4 g2w2 g2t256; do
  if [ "$v" = base ]; then unset LT_LIB_PATH; else export LT_LIB_PATH=$PWD/paper_1708_03183_b200/libltcuda_$v.so; fi
  for a in "2 --chains 10 --ts 32 --steps 10" "3 --ts 16,24,32,48 --steps 3" "4 4096 2048 --ts 12,16,24,32 --steps 3"; do
    timeout 600 python tools/sweep_ts.py $a 2>&1 | grep '"ts"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v [$a]', d.get('ts'), d.get('ms_per_step'), '%.4g'%d.get('value',0), d.get('wide'), d.get('smem'), d.get('error',''))"
  done
done > $O/ab.txt 2>&1
cat $O/ab.txt
