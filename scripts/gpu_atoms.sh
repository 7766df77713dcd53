#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -rf -k "sparse or c4 or paged or k8 or gather or residual or cluster or golden or oracle" > gpurun_out/atoms_pytest.txt 2>&1; echo "pytest rc $?" >> gpurun_out/atoms_pytest.txt
tail -3 gpurun_out/atoms_pytest.txt
for a in 0 1; do FB_GATHER_ATOMS=$a timeout 300 python scripts/exp_k8.py 0.1 0.2 0.3 0.5; done 2>&1 | tee gpurun_out/k8_atoms.txt
