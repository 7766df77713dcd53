#!/bin/bash
# session-4: K2 TMA-store bounds test (sentinel tail after the output)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_k2_store.py -m gpu -q -x > gpurun_out/s4j_pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s4j_pytest.txt
