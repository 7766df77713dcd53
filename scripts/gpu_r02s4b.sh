#!/bin/bash
# session-4: K2 v2 TMA-store epilogue -- parity tests, A/B, two-rank bench check
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_k2_store.py tests/test_partial_bf16.py -m gpu -q -x > gpurun_out/s4b_pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s4b_pytest.txt
timeout 300 python scripts/ab_k2_store.py 16 32 64 > gpurun_out/s4b_ab.txt 2>&1; echo "ab rc=$?"; cat gpurun_out/s4b_ab.txt | tail -12
FB_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --workload c3 --steps 3 --exchange nccl > gpurun_out/s4b_c3_2rank.json 2> gpurun_out/s4b_c3_2rank.err; echo "2rank rc=$?"; tail -1 gpurun_out/s4b_c3_2rank.json | cut -c1-300; tail -3 gpurun_out/s4b_c3_2rank.err
