# round 2, call f: plan statistics (smem per tile distribution), 256-thread variants, config-5 sweep
for a in "2 --chains 10 --ts 32 --steps 3" "3 --ts 24 --steps 3" "4 2048 1024 --ts 12,16 --steps 3"; do
  LT_DEBUG_PLAN=1 timeout 300 python tools/sweep_ts.py $a > gpurun_out/r02f_plan_$(echo $a | cut -c1).txt 2>&1
done
timeout 1800 bash tools/ab_variants.sh "base t256 t256b" "2 --chains 10 --ts 32 --steps 10" "3 --ts 24 --steps 3" "4 4096 2048 --ts 12,16 --steps 3" > gpurun_out/r02f_ab.txt 2>&1
timeout 2400 python tools/sweep_config5.py --out gpurun_out/r02f_config5.jsonl > gpurun_out/r02f_config5.log 2>&1
cat gpurun_out/r02f_ab.txt; grep "lt plan" gpurun_out/r02f_plan_*.txt | head -60
