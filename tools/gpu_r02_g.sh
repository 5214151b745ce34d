# round 2, call g: 128-register build at <= 4 CTAs/SM (A/B), partitioned path smoke, default bench line
timeout 1500 bash tools/ab_variants.sh "base w4" "3 --ts 16,24 --steps 3" "4 4096 2048 --ts 12,16 --steps 3" > gpurun_out/r02g_ab.txt 2>&1
timeout 900 python bench.py --config 3 --partitioned --steps 3 --warmup 2 > gpurun_out/r02g_part.json 2> gpurun_out/r02g_part.err
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/r02g_c4.json 2> gpurun_out/r02g_c4.err
cat gpurun_out/r02g_ab.txt gpurun_out/r02g_part.json gpurun_out/r02g_c4.json; tail -3 gpurun_out/r02g_part.err gpurun_out/r02g_c4.err
