P=paper_2602_05305_b200
for rnd in 1 2; do
for lib in libfb200_old.so libfb200.so; do
  FB_LIB_PATH=$PWD/$P/$lib timeout 300 python scripts/ab_c3b1.py
  FB_LIB_PATH=$PWD/$P/$lib timeout 300 python scripts/ab_vprod.py
done; done
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
