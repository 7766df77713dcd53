#!/bin/bash
# round-2 evidence pass: compute-sanitizer over the new kernels, ncu captures,
# secondary config lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
{
echo "== memcheck: cluster split-K K1 / K8 (cluster + atoms), bf16 partials"
timeout 1200 $S --tool memcheck python -m pytest tests/test_cluster_splitk.py tests/test_partial_bf16.py -m gpu -q -x 2>&1 | tail -3
echo "== racecheck: cluster split-K (one K1 shape, one K8 shape)"
timeout 1200 $S --tool racecheck python -m pytest tests/test_cluster_splitk.py -m gpu -q -x -k "8-128-16384 or sparse_cached_step and 0.1-True" 2>&1 | tail -3
echo "== synccheck: cluster split-K K8"
timeout 1200 $S --tool synccheck python -m pytest tests/test_cluster_splitk.py -m gpu -q -x -k "sparse_cached_step and 0.1-True" 2>&1 | tail -3
echo "== memcheck: K2 v1 / v2 / token-major with the bf16 cached partial"
timeout 1200 $S --tool memcheck python -m pytest tests/test_tokmajor.py tests/test_partial_bf16.py -m gpu -q -x -k "k2 or tokmajor" 2>&1 | tail -3
} > gpurun_out/sanitize_r02.txt 2>&1
cat gpurun_out/sanitize_r02.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:refresh_kernel -s 3 -c 1 -o gpurun_out/k8_cluster_atoms_r02 -f python scripts/trace_k8.py 0.1 > /dev/null 2>&1; echo "k8 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:refresh_kernel -s 9 -c 1 -o gpurun_out/k7_residual_r02 -f python scripts/exp_k7.py > /dev/null 2>&1; echo "k7 rc=$?"
timeout 2000 python scripts/bench_configs.py --out gpurun_out/r02_configs_final.jsonl > gpurun_out/r02_configs_final.log 2>&1; echo "configs rc=$?"
