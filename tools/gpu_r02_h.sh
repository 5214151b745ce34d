# round 2, call h: TMA gather4 build -- GPU tests, then TMA vs cp.async (LT_NO_TMA=1) A/B
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02h_pytest.log 2>&1
tail -3 gpurun_out/r02h_pytest.log
for rep in 1 2; do
 for mode in tma notma; do
  if [ $mode = notma ]; then export LT_NO_TMA=1; else unset LT_NO_TMA; fi
  for a in "2 --chains 10 --ts 32 --steps 10" "3 --ts 16 --steps 3" "4 4096 2048 --ts 12 --steps 3"; do
    timeout 600 python tools/sweep_ts.py $a 2>&1 | grep '"ts"' | sed "s/^/$mode rep$rep /"
  done
 done
done > gpurun_out/r02h_ab.txt 2>&1
cat gpurun_out/r02h_ab.txt | cut -c1-200
