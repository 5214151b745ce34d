#!/bin/bash
# usage (GPU box): make -C paper_1708_03183_b200/csrc all timing && bash tools/profile_all.sh
# Final-state evidence: bench lines (no profiler), launch list, ncu full capture of k_dataflow.
set -x
O=gpurun_out/prof
mkdir -p $O
python bench.py > $O/bench_c2.json 2> $O/bench_c2.err
python bench.py --config 3 --steps 5 > $O/bench_c3.json 2> $O/bench_c3.err
python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_dataflow -s 2 -c 1 -o $O/c2_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_c2.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:k_dataflow -c 1 -o $O/c3_full python bench.py --config 3 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/ncu_c3.log 2>&1
ls -la $O
export LT_LIB_PATH=$PWD/paper_1708_03183_b200/libltcuda_timing.so
for pad in 0 90; do echo "== phase timing config 2 ts 28, LT_SMEM_PAD_KB=$pad"; LT_SMEM_PAD_KB=$pad python tools/phase_timing.py 2 28; done > $O/phase_c2.txt 2>&1
for pad in 0; do echo "== phase timing config 3 ts 24, LT_SMEM_PAD_KB=$pad"; LT_SMEM_PAD_KB=$pad python tools/phase_timing.py 3 24; done > $O/phase_c3.txt 2>&1
