# compute-sanitizer over the r01g changes: token-major K2, the shuffle-broadcast
# split merge (multi-chunk items), 256-bit K1 / K2 stores
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
{
echo "== memcheck token-major K2"
timeout 900 $S --tool memcheck python -m pytest tests/test_tokmajor.py -q -x 2>&1 | tail -3
echo "== racecheck token-major K2 (one case)"
timeout 900 $S --tool racecheck python -m pytest tests/test_tokmajor.py -q -x -k "3-8-2-16" 2>&1 | tail -3
echo "== memcheck split merge (items over 148 CTAs, multi-segment) + K2 cached-step kernels"
timeout 1200 $S --tool memcheck python -m pytest tests/test_gpu_attention.py -q -x -k "stream_k_segments or cached_step_kernel_vs_oracle and 128-" 2>&1 | tail -3
echo "== memcheck sparse K7 / K8 (fused final merge)"
timeout 900 $S --tool memcheck python -m pytest tests/test_gpu_attention.py -q -x -k "sparse_partitioned_and_cached" 2>&1 | tail -3
} > gpurun_out/sanitize_r01g.txt 2>&1
cat gpurun_out/sanitize_r01g.txt
