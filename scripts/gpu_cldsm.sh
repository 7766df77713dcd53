#!/bin/bash
cd $GRAFT_REPO_ROOT
for d in 0 1 0 1; do echo "DSMEM=$d"; FB_K1_CLUSTER_DSMEM=$d timeout 300 python scripts/exp_k8.py 0.1 0.2; done
FB_K1_CLUSTER_DSMEM=1 CLUSTER_STAMPS=1 timeout 300 python scripts/trace_k8.py 0.1
FB_K1_CLUSTER_DSMEM=1 timeout 600 python -m pytest tests/test_cluster_splitk.py -m gpu -q -x 2>&1 | tail -2
