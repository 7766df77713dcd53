#!/bin/bash
cd $GRAFT_REPO_ROOT
for rep in 1 2; do for dg in 0 1 2; do FB_K8_DIAG=$dg timeout 300 python scripts/exp_k8.py 0.1 0.3 0.5; done; done
