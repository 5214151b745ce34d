# round 2: config-5 sweep (one rank's share) with the block layout pass, final build
mkdir -p gpurun_out/r02c5
timeout 3000 python tools/sweep_config5.py --layout block --out gpurun_out/r02c5/sweep_block.jsonl > gpurun_out/r02c5/sweep.log 2>&1
tail -5 gpurun_out/r02c5/sweep.log | cut -c1-300; wc -l gpurun_out/r02c5/sweep_block.jsonl
