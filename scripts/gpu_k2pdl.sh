#!/bin/bash
# A/B: K2 signalling its dependent launch right after the PDL wait (A) vs after its Q/K/V landed (B)
cd $GRAFT_REPO_ROOT
P=paper_2602_05305_b200
cp $P/libfb200.so $P/libfb200_A.so; cp $P/libfb200.so $P/libfb200_B.so
for b in 16 4 32; do AB_EXTB=1 timeout 300 python scripts/ab_k2.py $PWD/$P/libfb200_A.so $PWD/$P/libfb200_B.so $b FB_K2_PDL_LATE=0 FB_K2_PDL_LATE=1 2>&1 | tail -2; done
