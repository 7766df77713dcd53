for rnd in 1 2; do for p in 0 4 3 2; do FB_K5_POLY=$p timeout 300 python scripts/ab_k5.py; done; done
FB_K5_POLY=2 timeout 600 python -m pytest tests/test_gpu_attention.py -q -x -k "mass or sparse" 2>&1 | tail -2
