#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/var_pytest.txt 2>&1; echo "pytest rc $?" >> gpurun_out/var_pytest.txt
tail -2 gpurun_out/var_pytest.txt
python scripts/exp_k7.py; FB_K1_CLUSTER=0 python scripts/exp_k7.py; FB_GATHER_ATOMS=0 FB_K1_CLUSTER=0 python scripts/exp_k7.py
python scripts/exp_k8.py 0.1 0.2 0.3 0.5; FB_K1_CLUSTER=0 python scripts/exp_k8.py 0.1 0.2 0.3 0.5
python scripts/ab_cluster.py 2>&1 | grep "C2 b=4\|b=1 P=8\|b=1 P=1"
