mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_attention.py tests/test_pair.py tests/test_prefill.py -x -q 2>&1 | tail -2
for rnd in 1 2; do for vp in 1 0; do FB_K1_VPROD=$vp timeout 300 python scripts/ab_vprod.py; done; done
