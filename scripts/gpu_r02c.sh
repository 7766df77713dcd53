#!/bin/bash
# round 2 re-entry check: full GPU suite (incl. the fixed reference suites), smoke, bench, C3 anchor
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf --durations=15 > gpurun_out/r02c_pytest.txt 2>&1
echo "pytest rc $?" >> gpurun_out/r02c_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c_smoke.txt 2>&1
echo "smoke rc $?" >> gpurun_out/r02c_smoke.txt
timeout 600 python bench.py > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err
echo "bench rc $?" >> gpurun_out/r02c_bench.err
