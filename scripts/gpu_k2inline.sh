P=paper_2602_05305_b200
cp $P/libfb200.so /tmp/libA.so; cp $P/libfb200.so /tmp/libB.so
for b in 16 4 32; do timeout 300 python scripts/ab_k2.py /tmp/libA.so /tmp/libB.so $b FB_K2_INLINE=0 FB_K2_INLINE=1 2>&1 | tail -2; done
FB_K2_INLINE=1 timeout 600 python -m pytest tests/test_gpu_attention.py tests/test_graph_replay.py tests/test_counters.py -x -q 2>&1 | tail -2
