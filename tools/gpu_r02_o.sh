# round 2, call o: TMA scaffolding compiled out, per-tile record chunks, grouped-item masks
O=gpurun_out/r02o
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_dg.py tests/test_gpu_bench_parity.py tests/test_gpu_executor.py tests/test_gpu_distributed.py -x -q > $O/pytest.log 2>&1; tail -3 $O/pytest.log
run() {  # variant, env assignments..., then sweeps
  v=$1; shift
  if [ "$v" = base ]; then unset LT_LIB_PATH; else export LT_LIB_PATH=$PWD/paper_1708_03183_b200/libltcuda_$v.so; fi
  for a in "2 --chains 10 --ts 32 --steps 10" "3 --ts 16,24 --steps 3" "4 4096 2048 --ts 12,16 --steps 3"; do
    timeout 600 python tools/sweep_ts.py $a 2>&1 | grep '"ts"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v $LT_UNIFORM_CHUNKS [$a]', d.get('ts'), d.get('ms_per_step'), '%.4g'%d.get('value',0), d.get('wide'), d.get('smem'), d.get('error',''))"
  done
}
for v in g0 base g13 g5 g8 b4; do run $v; done > $O/ab.txt 2>&1
export LT_UNIFORM_CHUNKS=1; for v in g0 base; do run $v; done >> $O/ab.txt 2>&1; unset LT_UNIFORM_CHUNKS
cat $O/ab.txt
for v in t0 t15; do
  export LT_LIB_PATH=$PWD/paper_1708_03183_b200/libltcuda_$v.so
  echo "== $v"; timeout 600 python tools/phase_timing.py 4 12 2048 1024 2>&1 | tail -14
  echo "== $v"; timeout 600 python tools/phase_timing.py 3 16 2>&1 | tail -14
done > $O/phase.txt 2>&1
cat $O/phase.txt
