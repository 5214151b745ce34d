# round 2, call m: grouped DG items (cell x row-group, facet x point-group) -- parity, A/B, phase timing
O=gpurun_out/r02m
mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_dg.py tests/test_gpu_bench_parity.py tests/test_gpu_executor.py -x -q > $O/pytest.log 2>&1; tail -3 $O/pytest.log
timeout 1500 bash tools/ab_variants.sh "base nogroup" "2 --chains 10 --ts 32 --steps 10" "3 --ts 16,24 --steps 3" "4 4096 2048 --ts 12,16 --steps 3" > $O/ab.txt 2>&1
cat $O/ab.txt
export LT_LIB_PATH=$PWD/paper_1708_03183_b200/libltcuda_timing.so
LT_DEBUG_PLAN=1 timeout 600 python tools/phase_timing.py 4 12 2048 1024 > $O/phase_c4.txt 2>&1
LT_DEBUG_PLAN=1 timeout 600 python tools/phase_timing.py 3 16 > $O/phase_c3.txt 2>&1
cat $O/phase_c4.txt $O/phase_c3.txt
