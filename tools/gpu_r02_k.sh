# round 2, call k: control A/B (current build vs the call-h build 3a39c8e without TMA), clocks
export LT_NO_TMA=1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,power.limit,clocks_event_reasons.active --format=csv > gpurun_out/r02k_smi.txt
timeout 1500 bash tools/ab_variants.sh "base h" "2 --chains 10 --ts 32 --steps 10" "3 --ts 16 --steps 3" "4 4096 2048 --ts 12 --steps 3" > gpurun_out/r02k_ab.txt 2>&1
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-omega > gpurun_out/r02k_c3.json 2>&1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,power.limit,clocks_event_reasons.active --format=csv >> gpurun_out/r02k_smi.txt
cat gpurun_out/r02k_ab.txt gpurun_out/r02k_smi.txt; tail -c 600 gpurun_out/r02k_c3.json
