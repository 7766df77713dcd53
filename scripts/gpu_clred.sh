#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -rf -k "sparse or c4 or paged or k8 or gather or residual or cluster or golden or oracle" > gpurun_out/clred_pytest.txt 2>&1; echo "pytest rc $?" >> gpurun_out/clred_pytest.txt
tail -3 gpurun_out/clred_pytest.txt
timeout 300 python scripts/exp_k8.py 0.1 0.2 0.3 0.5
timeout 300 python scripts/trace_k8.py 0.1
timeout 600 python scripts/ab_cluster.py 2>&1 | grep "C2 b=4\|P=8"
