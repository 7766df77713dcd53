#!/bin/bash
# session-4: V-split barrier in K2 v1 / token-major, Q/K half barriers in v2 -- parity + A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_k2_store.py tests/test_partial_bf16.py tests/test_gpu_attention.py tests/test_tokmajor.py tests/test_replay.py tests/test_engine_paths.py tests/test_capi.py -m gpu -q -x > gpurun_out/s4e_pytest.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s4e_pytest.txt
timeout 300 python scripts/ab_k2_store.py 4 16 32 64 > gpurun_out/s4e_ab.txt 2>&1; echo "ab rc=$?"; cat gpurun_out/s4e_ab.txt | tail -20
