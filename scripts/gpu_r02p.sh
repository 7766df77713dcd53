#!/bin/bash
# full GPU suite, smoke, default bench, secondary config lines (K5 fused, C1 drop-in host path)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r02p_pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02p_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02p_smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02p_smoke.txt
timeout 900 python bench.py > gpurun_out/r02p_bench.json 2> gpurun_out/r02p_bench.err; echo "bench rc=$?"; tail -1 gpurun_out/r02p_bench.json | cut -c1-200
timeout 2000 python scripts/bench_configs.py --out gpurun_out/r02p_configs.jsonl > gpurun_out/r02p_configs.log 2>&1; echo "configs rc=$?"
