mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:internal_merge -s 2 -c 1 -o gpurun_out/k2_b16_r01f -f python scripts/profile_k1.py --batch 16 --layers 2 --reps 2 > gpurun_out/ncu_k2_r01f.log 2>&1; echo "k2 rc=$?"
