#!/bin/bash
# round-2 ncu evidence (summaries copied to profiles/ afterwards)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'refresh|internal_merge|combine|partial_simt|pair_kernel|quad' -c 1300 --csv --log-file gpurun_out/launches_r02.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-sweep > gpurun_out/ncu_launches_r02.log 2>&1; echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:refresh_kernel -s 2 -c 1 -o gpurun_out/k1_b32_r02 -f python scripts/profile_k1.py --batch 32 --layers 2 --reps 2 > gpurun_out/ncu_k1_r02.log 2>&1; echo "k1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:internal_merge_v2 -s 2 -c 1 -o gpurun_out/k2v2_b32_r02 -f python scripts/profile_k1.py --batch 32 --layers 2 --reps 2 > gpurun_out/ncu_k2_r02.log 2>&1; echo "k2 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:refresh_kernel -s 3 -c 1 -o gpurun_out/k8_cluster10_r02 -f python scripts/trace_k8.py 0.1 > gpurun_out/ncu_k8_r02.log 2>&1; echo "k8 rc=$?"
for f in k1_b32_r02 k2v2_b32_r02 k8_cluster10_r02; do ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/$f.raw.csv 2>/dev/null; done
echo done
