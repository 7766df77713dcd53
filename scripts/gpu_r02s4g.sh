#!/bin/bash
# session-4: ncu of the new K2 v2 (b=32, TMA store + split barriers) and the bench launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:internal_merge_v2 -s 4 -c 1 -o gpurun_out/s4g_k2v2_b32 -f python scripts/profile_k1.py --batch 32 --layers 2 --reps 2 > gpurun_out/s4g_ncu_k2.log 2>&1; echo "k2 rc=$?"; tail -3 gpurun_out/s4g_ncu_k2.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s4g_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-sweep > gpurun_out/s4g_bench_ncu.log 2>&1; echo "ncu rc=$?"
