# round 2, call x (re-run as r02x2 after the work-item masks changed): FINAL-build evidence (block layout pass, 4 KB first-pass scratch): full GPU test suite,
# bench lines (no profiler), launch lists, ncu --set full of the config 4 / 3 / 2 bench launches, phase cycles
O=gpurun_out/r02x2
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; tail -3 $O/pytest_gpu.log
python -c 'import __graft_entry__ as g; g.smoke()' > $O/smoke.log 2>&1; tail -1 $O/smoke.log
timeout 900 python bench.py > $O/bench_c4.json 2> $O/bench_c4.err; tail -c 400 $O/bench_c4.json
timeout 600 python bench.py --config 3 --stated-ts --steps 5 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 300 python bench.py --config 2 > $O/bench_c2.json 2> $O/bench_c2.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_ref.json 2> $O/bench_ref.err
for c in 4 3 2; do
timeout 900 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-omega > $O/plain_c$c.json 2> $O/plain_c$c.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_dataflow|k_pack_ro|FillFunctor' -c 40 --csv --log-file $O/launches_c$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-omega > $O/ncu_launch_c$c.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_dataflow -s 3 -c 1 -o $O/c${c}_full python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-omega > $O/ncu_c$c.log 2>&1
python tools/ncu_extract.py $O/c${c}_full.ncu-rep $O/ncu_c$c > /dev/null 2>&1; rm -f $O/c${c}_full.ncu-rep
done
export LT_LIB_PATH=$PWD/paper_1708_03183_b200/libltcuda_timing.so
timeout 600 python tools/phase_timing.py 4 24 2048 1024 2>&1 | tail -14 > $O/phase_c4.txt
timeout 600 python tools/phase_timing.py 3 32 2>&1 | tail -14 > $O/phase_c3.txt
unset LT_LIB_PATH
cat $O/phase_c4.txt $O/phase_c3.txt
ls -la $O
