#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -k "sparse or c4 or paged or k8 or gather or residual or partial_bf16 or large" > gpurun_out/k8fin_pytest.txt 2>&1; echo "pytest rc $?" >> gpurun_out/k8fin_pytest.txt
tail -3 gpurun_out/k8fin_pytest.txt
for rep in 1 2; do for dg in 0 3; do FB_K8_DIAG=$dg timeout 300 python scripts/exp_k8.py 0.1 0.2 0.3 0.5; done; done
