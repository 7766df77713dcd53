P=paper_2602_05305_b200
for b in 16 4 32; do timeout 300 python scripts/ab_k2.py $PWD/$P/libfb200_A.so $PWD/$P/libfb200_B.so $b FB_K2_V2=0 FB_K2_V2=0 2>&1 | tail -2; done
