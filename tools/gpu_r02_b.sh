# round 2, call b: GPU tests incl. full-size parity, bench configs 4/3/2
free -g > gpurun_out/r02b_free.txt; nvidia-smi >> gpurun_out/r02b_free.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02b_pytest.log 2>&1
tail -5 gpurun_out/r02b_pytest.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r02b_c4.json 2> gpurun_out/r02b_c4.err
timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --stated-ts > gpurun_out/r02b_c3.json 2> gpurun_out/r02b_c3.err
timeout 300 python bench.py --config 2 --steps 10 --warmup 3 > gpurun_out/r02b_c2.json 2> gpurun_out/r02b_c2.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 2 > gpurun_out/r02b_ref.json 2> gpurun_out/r02b_ref.err
tail -c 3000 gpurun_out/r02b_c4.err
