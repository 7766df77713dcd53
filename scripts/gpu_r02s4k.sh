#!/bin/bash
# session-4 snapshot of every secondary config line on the final build
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 2400 python scripts/bench_configs.py --out gpurun_out/s4k_configs.jsonl > gpurun_out/s4k_configs.log 2>&1; echo "configs rc=$?"; tail -5 gpurun_out/s4k_configs.log
