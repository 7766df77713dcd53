timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:score_kernel -s 2 -c 2 -o gpurun_out/k5_full python scripts/profile_sparse.py > gpurun_out/ncu_k5.log 2>&1; echo "ncu-k5 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:refresh_kernel -s 4 -c 2 -o gpurun_out/k78_full python scripts/profile_sparse.py > gpurun_out/ncu_k78.log 2>&1; echo "ncu-k78 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:internal_merge -s 2 -c 1 -o gpurun_out/k2_full python scripts/profile_k1.py --batch 8 --layers 3 > gpurun_out/ncu_k2.log 2>&1; echo "ncu-k2 rc=$?"
