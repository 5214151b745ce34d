# round 2: config-5 sweep (one rank's share) with the block layout pass, final build;
# one process per (degree, chain length): every point rebuilds the problem in its layout
mkdir -p gpurun_out/r02c5
rm -f gpurun_out/r02c5/sweep_block.jsonl
for p in 1 2 3 4; do for T in 1 2 4; do
  timeout 900 python tools/sweep_config5.py --layout block --degrees $p --chains $T --out gpurun_out/r02c5/sweep_block.jsonl >> gpurun_out/r02c5/sweep.log 2>&1
done; done
wc -l gpurun_out/r02c5/sweep_block.jsonl; grep -c error gpurun_out/r02c5/sweep_block.jsonl
