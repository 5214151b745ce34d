# round 2, call w: more block shapes; full-size config 4 for the best two
O=gpurun_out/r02w
mkdir -p $O
sw() { timeout 900 python tools/sweep_ts.py "$@" 2>&1 | grep -E '"ts"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(' '.join(sys.argv[1:]), '|', d.get('ts'), d.get('ms_per_step'), '%.4g'%d.get('value',0), d.get('wide'), d.get('smem'), d.get('colors'), d.get('plan_s'), d.get('gpu_used_gb'), d.get('error',''))" "$@"; }
{
sw 4 --ts 24 --steps 3 --renumber block:4x3
sw 4 --ts 16 --steps 3 --renumber block:4x2
sw 4 4096 2048 --ts 24 --steps 3 --renumber block:3x4
sw 4 4096 2048 --ts 24 --steps 3 --renumber block:6x2
sw 4 4096 2048 --ts 24 --steps 3 --renumber block:2x6
sw 4 4096 2048 --ts 16 --steps 3 --renumber block:2x4
sw 4 4096 2048 --ts 16 --steps 3 --renumber block:8x1
sw 4 4096 2048 --ts 28 --steps 3 --renumber block:7x2
sw 4 4096 2048 --ts 20 --steps 3 --renumber block:2x5
sw 3 --ts 32 --steps 3 --renumber block:8x2
sw 3 --ts 32 --steps 3 --renumber block:2x8
sw 3 --ts 40 --steps 3 --renumber block:4x5
sw 3 --ts 28 --steps 3 --renumber block:7x2
sw 3 --ts 36 --steps 3 --renumber block:3x6
sw 3 --ts 24 --steps 3 --renumber block:3x4
} > $O/sweep.txt 2>&1
cat $O/sweep.txt
