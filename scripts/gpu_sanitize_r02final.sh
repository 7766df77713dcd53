#!/bin/bash
# compute-sanitizer over this session's late kernel changes: the K1-epilogue
# final merge (fin_whole, merge launch skipped), the top-k early exit / global
# keys, the fused K5
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
{
echo "== memcheck: K1 epilogue final merge, top-k, fused K5"
timeout 1200 $S --tool memcheck python -m pytest tests/test_quad.py tests/test_topk.py tests/test_k5_fused.py -m gpu -q -x -k "final_merge or topk or fused_mass_equals" 2>&1 | tail -3
echo "== racecheck: top-k (shared-memory histogram, candidate ranking)"
timeout 1200 $S --tool racecheck python -m pytest tests/test_topk.py -m gpu -q -x -k "groups1 or 1]" 2>&1 | tail -3
echo "== racecheck: K1 epilogue final merge"
timeout 1200 $S --tool racecheck python -m pytest tests/test_quad.py -m gpu -q -x -k "final_merge and True" 2>&1 | tail -3
} > gpurun_out/sanitize_r02final.txt 2>&1
cat gpurun_out/sanitize_r02final.txt
