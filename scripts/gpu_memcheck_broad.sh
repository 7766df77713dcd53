#!/bin/bash
# compute-sanitizer memcheck over the broad GPU suites of the final build
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
for f in test_gpu_attention test_quad test_cluster_splitk test_partial_bf16 test_paged test_tokmajor test_k5_fused test_topk test_dropin_host test_engine_paths test_prefill; do
  echo "== $f"
  timeout 900 $S --tool memcheck --print-limit 5 python -m pytest tests/$f.py -m gpu -q -x 2>&1 | grep -E "passed|failed|ERROR SUMMARY|Invalid|error" | head -4
done > gpurun_out/memcheck_broad.txt 2>&1
cat gpurun_out/memcheck_broad.txt
