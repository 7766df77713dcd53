#!/bin/bash
# session-4: bench launch list (our kernels only: the KV initialisation kernels fill the first 400 launches otherwise)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'refresh|internal_merge|combine|merge|partial' -c 1200 --csv --log-file gpurun_out/s4h_bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-sweep > gpurun_out/s4h_bench_ncu.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/s4h_bench_ncu.log
