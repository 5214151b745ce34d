# round 2, call i: TMA gather4 (128-byte aligned, padded rows) -- tests, A/B vs cp.async, 5 CTAs/SM variant
timeout 1200 python -m pytest tests/test_gpu_dg.py tests/test_gpu_bench_parity.py -x -q > gpurun_out/r02j_pytest.log 2>&1
tail -3 gpurun_out/r02j_pytest.log
for rep in 1 2; do
 for mode in tma notma w5; do
  unset LT_NO_TMA LT_LIB_PATH
  if [ $mode = notma ]; then export LT_NO_TMA=1; fi
  if [ $mode = w5 ]; then export LT_LIB_PATH=$PWD/paper_1708_03183_b200/libltcuda_w5.so; fi
  for a in "2 --chains 10 --ts 32 --steps 10" "3 --ts 12,16 --steps 3" "4 4096 2048 --ts 10,12 --steps 3"; do
    timeout 300 python tools/sweep_ts.py $a 2>&1 | grep '"ts"' | sed "s/^/$mode rep$rep /"
  done
 done
done > gpurun_out/r02j_ab.txt 2>&1
cut -c1-150 gpurun_out/r02j_ab.txt
