# round 2, call t: field-lane volume items (operator tables as constant-bank operands): parity, A/B, phase cycles
O=gpurun_out/r02t
mkdir -p $O
export LT_LIB_PATH=$PWD/paper_1708_03183_b200/libltcuda_vf.so
timeout 1500 python -m pytest tests/test_gpu_chunks.py tests/test_gpu_dg.py tests/test_gpu_bench_parity.py tests/test_gpu_executor.py -x -q > $O/pytest_vf.log 2>&1; tail -3 $O/pytest_vf.log
unset LT_LIB_PATH
for rep in 1 2; do
for v in base vf; do
  if [ "$v" = base ]; then unset LT_LIB_PATH; else export LT_LIB_PATH=$PWD/paper_1708_03183_b200/libltcuda_$v.so; fi
  for a in "2 --chains 10 --ts 32 --steps 10" "3 --ts 32 --steps 5" "4 4096 2048 --ts 16 --steps 5"; do
    timeout 600 python tools/sweep_ts.py $a 2>&1 | grep '"ts"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v rep$rep [$a]', d.get('ts'), d.get('ms_per_step'), '%.4g'%d.get('value',0), d.get('wide'), d.get('smem'), d.get('error',''))"
  done
done
done > $O/ab.txt 2>&1
cat $O/ab.txt
export LT_LIB_PATH=$PWD/paper_1708_03183_b200/libltcuda_vft.so
timeout 600 python tools/phase_timing.py 4 16 2048 1024 2>&1 | tail -14 > $O/phase_c4_vf.txt
timeout 600 python tools/phase_timing.py 3 32 2>&1 | tail -14 > $O/phase_c3_vf.txt
unset LT_LIB_PATH
cat $O/phase_c4_vf.txt $O/phase_c3_vf.txt
