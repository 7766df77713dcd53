#!/bin/bash
# session-4: K2 v2 register cap A/B across two library builds (FB_LIB_PATH):
# base = __launch_bounds__(288, 2) (96 registers, 4-20 B spills), maxnreg = __maxnreg__(112) (no spills)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
  for v in base maxnreg; do
    echo "== $v ($i)"
    FB_LIB_PATH=$GRAFT_REPO_ROOT/build_ab/libfb200_$v.so timeout 300 python scripts/ab_k2_store.py 16 32 64 2>&1 | grep -E "default|equal"
  done
done > gpurun_out/s4l_ab.txt 2>&1
cat gpurun_out/s4l_ab.txt
