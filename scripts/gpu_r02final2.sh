#!/bin/bash
# end-of-session snapshot: full GPU suite, smoke, bench, every secondary config line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/r02final2_pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02final2_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02final2_smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02final2_smoke.txt
timeout 900 python bench.py > gpurun_out/r02final2_bench.json 2> gpurun_out/r02final2_bench.err; echo "bench rc=$?"; tail -1 gpurun_out/r02final2_bench.json | cut -c1-200
timeout 2400 python scripts/bench_configs.py --out gpurun_out/r02final2_configs.jsonl > gpurun_out/r02final2_configs.log 2>&1; echo "configs rc=$?"
