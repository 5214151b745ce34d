# round 2, call c: P3 T=2 seed-tile sweep at growing sizes (memory + speed), wide test fix
timeout 600 python -m pytest tests/test_gpu_dg.py tests/test_gpu_bench_parity.py tests/test_gpu_inspector.py -x -q > gpurun_out/r02c_pytest.log 2>&1
tail -3 gpurun_out/r02c_pytest.log
timeout 600 python tools/sweep_ts.py 4 1024 512 --ts 8,12,16,20,24,32 > gpurun_out/r02c_sweep_small.jsonl 2>&1
timeout 900 python tools/sweep_ts.py 4 4096 2048 --ts 12,16 > gpurun_out/r02c_sweep_mid.jsonl 2>&1
timeout 900 python tools/sweep_ts.py 4 --ts 16 > gpurun_out/r02c_sweep_full.jsonl 2>&1
cat gpurun_out/r02c_sweep_*.jsonl
