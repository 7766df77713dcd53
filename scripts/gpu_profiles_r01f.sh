#!/bin/bash
# ncu evidence for the r01f kernels (summaries copied to profiles/ afterwards).
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'refresh|internal_merge|combine|partial_simt|pair_kernel' -c 2500 --csv --log-file gpurun_out/launches_r01f.csv python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:refresh_kernel -s 2 -c 1 -o gpurun_out/k1_b16_r01f -f python scripts/profile_k1.py --batch 16 --layers 2 --reps 2 > gpurun_out/ncu_k1.log 2>&1; echo "k1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:pair_kernel -c 1 -o gpurun_out/pair_prefill_r01f -f python scripts/prof_pair.py pair prefill > gpurun_out/ncu_pairpf.log 2>&1; echo "pair prefill rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:refresh_kernel -c 1 -o gpurun_out/single_prefill_r01f -f python scripts/prof_pair.py single prefill > gpurun_out/ncu_singlepf.log 2>&1; echo "single prefill rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:internal_merge_v2 -s 2 -c 1 -o gpurun_out/k2v2_b32_r01f -f python scripts/profile_k1.py --batch 32 --layers 2 --reps 2 > gpurun_out/ncu_k2v2.log 2>&1; echo "k2v2 rc=$?"
