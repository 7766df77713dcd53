CUDA_LAUNCH_BLOCKING=1 timeout 300 python scripts/debug_k2.py 2>&1 | tail -5
timeout 600 compute-sanitizer --tool memcheck python scripts/debug_k2.py 2>&1 | head -40
