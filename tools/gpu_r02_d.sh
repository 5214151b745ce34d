# round 2, call d: default bench (config 4) line, launch list + dram traffic of the exact bench
# kernel, ncu full capture of k_dataflow on a config-4 cut (P3 T=2 ts 16, 1024x512)
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02d_c4.json 2> gpurun_out/r02d_c4.err
A="--steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-omega"
timeout 600 python bench.py $A > gpurun_out/r02d_plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02d_launches_c4.csv python bench.py $A > gpurun_out/r02d_ncu_launch.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_dataflow -s 1 -c 1 --csv --log-file gpurun_out/r02d_traffic_c4.csv python bench.py $A > gpurun_out/r02d_ncu_traffic.log 2>&1
timeout 300 python tools/sweep_ts.py 4 1024 512 --ts 16 --steps 1 > gpurun_out/r02d_cut_plain.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_dataflow -s 2 -c 1 -o gpurun_out/r02d_c4cut python tools/sweep_ts.py 4 1024 512 --ts 16 --steps 1 > gpurun_out/r02d_ncu_full.log 2>&1
ls -la gpurun_out
