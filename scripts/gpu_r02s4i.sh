#!/bin/bash
# session-4: K2 v2 early O_ext register read -- parity + A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_k2_store.py tests/test_partial_bf16.py -m gpu -q -x > gpurun_out/s4i_pytest.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s4i_pytest.txt
timeout 300 python scripts/ab_k2_store.py 16 32 64 > gpurun_out/s4i_ab.txt 2>&1; echo "ab rc=$?"; grep -v "equal: True" gpurun_out/s4i_ab.txt | tail -20
