timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 900 python bench.py --steps 20 --warmup 3 --no-cpu > gpurun_out/bench.log 2>&1; echo "bench rc=$?"
timeout 600 python scripts/exp_k1_footprint.py
timeout 900 python scripts/bench_configs.py --only c5,c4 2>&1 | grep -E "C5|0.2,|0.1," | cut -c1-330
timeout 300 python scripts/trace_k1.py 8
