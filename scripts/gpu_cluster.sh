#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_cluster_splitk.py -m gpu -q -rf -x > gpurun_out/cl_pytest.txt 2>&1; echo "cl pytest rc $?" >> gpurun_out/cl_pytest.txt
tail -3 gpurun_out/cl_pytest.txt
timeout 600 python scripts/ab_cluster.py 2>&1 | tee gpurun_out/ab_cluster.txt
for dg in 0 2; do FB_K1_CLUSTER=$dg timeout 300 python scripts/exp_k8.py 0.1 0.3 0.5; done 2>&1 | tee gpurun_out/k8_cluster.txt
timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/cl_full_pytest.txt 2>&1; echo "full pytest rc $?" >> gpurun_out/cl_full_pytest.txt
tail -3 gpurun_out/cl_full_pytest.txt
