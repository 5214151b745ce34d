set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r02a_pytest.log
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/r02a_c2.json 2> gpurun_out/r02a_c2.err
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02a_c3.json 2> gpurun_out/r02a_c3.err
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --untiled > gpurun_out/r02a_c3u.json 2> gpurun_out/r02a_c3u.err
timeout 900 python bench.py --config 3 --ts 4096 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02a_c3ts4096.json 2> gpurun_out/r02a_c3ts4096.err
lscpu | head -20 > gpurun_out/r02a_lscpu.txt; nproc >> gpurun_out/r02a_lscpu.txt
