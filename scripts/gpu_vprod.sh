for rnd in 1 2; do for vp in 1 2; do FB_K1_VPROD=$vp timeout 300 python scripts/ab_vprod.py; done; done
FB_K1_VPROD=2 timeout 600 python -m pytest tests/test_gpu_attention.py tests/test_full_size.py -x -q -k "sparse or c4" 2>&1 | tail -2
