#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:refresh_kernel -s 2 -c 1 -o gpurun_out/k1_b16 python scripts/profile_k1.py --batch 16 --layers 2 --reps 2 > gpurun_out/ncu_k1.log 2>&1; echo "k1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:internal_merge -s 2 -c 1 -o gpurun_out/k2_b16 python scripts/profile_k1.py --batch 16 --layers 2 --reps 2 > gpurun_out/ncu_k2.log 2>&1; echo "k2 rc=$?"
