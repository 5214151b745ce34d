# round 2, call p: default build (LT_GROUPED per family, per-tile chunks, no TMA scaffolding):
# tests, Morton (Z-curve) cell renumbering vs row-major numbering, full-size config 4
O=gpurun_out/r02p
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_chunks.py tests/test_gpu_dg.py tests/test_gpu_bench_parity.py -x -q > $O/pytest.log 2>&1; tail -3 $O/pytest.log
sw() { timeout 900 python tools/sweep_ts.py $@ 2>&1 | grep -E '"ts"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('[$*]', d.get('ts'), d.get('ms_per_step'), '%.4g'%d.get('value',0), 'frac %.4f'%d.get('frac',0), d.get('wide'), d.get('smem'), d.get('tiles'), d.get('colors'), d.get('plan_s'), d.get('gpu_used_gb'), d.get('error',''))"; }
{
sw 3 --ts 16,24 --steps 3
sw 3 --ts 16,24,32 --steps 3 --renumber morton
sw 4 4096 2048 --ts 12,16 --steps 3
sw 4 4096 2048 --ts 8,12,16,24,32 --steps 3 --renumber morton
sw 4 --ts 12,16 --steps 3
sw 4 --ts 16,32 --steps 3 --renumber morton
} > $O/sweep.txt 2>&1
cat $O/sweep.txt
