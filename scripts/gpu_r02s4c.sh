#!/bin/bash
# session-4: K2 v2 V-split barrier A/B, PCIe ceiling, bench with the new K2 defaults
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_k2_store.py tests/test_partial_bf16.py tests/test_gpu_attention.py -m gpu -q -x > gpurun_out/s4c_pytest.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s4c_pytest.txt
timeout 300 python scripts/ab_k2_store.py 32 64 > gpurun_out/s4c_ab.txt 2>&1; echo "ab rc=$?"; cat gpurun_out/s4c_ab.txt | tail -10
timeout 120 python scripts/micro_pcie.py > gpurun_out/s4c_pcie.txt 2>&1; echo "pcie rc=$?"; cat gpurun_out/s4c_pcie.txt
timeout 900 python bench.py --no-cpu > gpurun_out/s4c_bench.json 2> gpurun_out/s4c_bench.err; echo "bench rc=$?"; tail -1 gpurun_out/s4c_bench.json | cut -c1-200
