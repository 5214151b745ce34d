# round 2, call z: partitioned path at N=1 with its own seed tile; P2 work-item masks at the final configuration
O=gpurun_out/r02z
mkdir -p $O
timeout 600 python bench.py --partitioned --steps 3 --warmup 3 --no-e2e > $O/bench_c4_partitioned_n1.json 2> $O/bench_c4_partitioned_n1.err; tail -c 300 $O/bench_c4_partitioned_n1.json
for rep in 1 2; do
for v in base m8 m9 m12 m0; do
  if [ "$v" = base ]; then unset LT_LIB_PATH; else export LT_LIB_PATH=$PWD/paper_1708_03183_b200/libltcuda_$v.so; fi
  for a in "3 --ts 32 --steps 5" "4 4096 2048 --ts 24 --steps 5"; do
    timeout 600 python tools/sweep_ts.py $a 2>&1 | grep '"ts"' | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print('$v rep$rep [$a]', d.get('ts'), d.get('ms_per_step'), '%.4g'%d.get('value',0), d.get('wide'), d.get('smem'), d.get('error',''))"
  done
done
done > $O/ab.txt 2>&1
cat $O/ab.txt
