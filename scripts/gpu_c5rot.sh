#!/bin/bash
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
timeout 300 python scripts/exp_c5.py
FB_K1_QUAD=1 timeout 300 python scripts/exp_c5.py
FB_K1_QUAD=1 FB_QUAD_ROT=0 timeout 300 python scripts/exp_c5.py
done
timeout 600 python -m pytest tests/test_quad.py tests/test_pair.py -m gpu -q -x 2>&1 | tail -2
timeout 300 python scripts/exp_k7.py
FB_GATHER_ATOMS=0 timeout 300 python scripts/exp_k7.py
FB_K1_CLUSTER=0 timeout 300 python scripts/exp_k7.py
FB_GATHER_ATOMS=0 FB_K1_CLUSTER=0 timeout 300 python scripts/exp_k7.py
