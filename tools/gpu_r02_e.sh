timeout 2400 bash tools/ab_variants.sh "base novec nores r01" "2 --chains 10 --ts 32 --steps 10" "3 --ts 24 --steps 3" "4 4096 2048 --ts 12,16 --steps 3" > gpurun_out/r02e_ab.txt 2>&1
cat gpurun_out/r02e_ab.txt
