#!/bin/bash
# Round measurement: bench (ours + reference arm), config lines, ncu launch list
# of the bench, ncu --set full of the top kernels.  Outputs in gpurun_out/.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench.log | cut -c1-300
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo "benchref rc=$?"
timeout 1500 python scripts/bench_configs.py --out gpurun_out/configs.jsonl > gpurun_out/configs.log 2>&1; echo "configs rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_launches.log 2>&1; echo "launches rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:refresh_kernel -s 2 -c 1 -o gpurun_out/k1_b16 python scripts/profile_k1.py --batch 16 --layers 2 --reps 2 > gpurun_out/ncu_k1.log 2>&1; echo "k1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:internal_merge -s 2 -c 1 -o gpurun_out/k2_b16 python scripts/profile_k1.py --batch 16 --layers 2 --reps 2 > gpurun_out/ncu_k2.log 2>&1; echo "k2 rc=$?"
