# round 2, call s: scheduling-independence (race) test, ncu captures of the config 3 and config 2 bench launches
O=gpurun_out/r02s
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_chunks.py tests/test_gpu_dg.py -x -q > $O/pytest.log 2>&1; tail -3 $O/pytest.log
for c in 3 2; do
timeout 600 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-omega > $O/plain_c$c.json 2> $O/plain_c$c.err && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dataflow -s 3 -c 1 -o $O/c${c}_full python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-omega > $O/ncu_c$c.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_dataflow|k_pack_ro|FillFunctor' -c 40 --csv --log-file $O/launches_c$c.csv python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-omega > $O/ncu_launch_c$c.log 2>&1
done
ls -la $O
