timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
FB_NO_PDL=1 timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_nopdl.log 2>&1; echo "bench-nopdl rc=$?"
timeout 600 python scripts/exp_k1_footprint.py 2>&1 | head -4
