#!/bin/bash
# session-3 entry check: full GPU suite + smoke + default bench on HEAD
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/r02o_pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02o_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02o_smoke.txt 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r02o_smoke.txt
timeout 900 python bench.py > gpurun_out/r02o_bench.json 2> gpurun_out/r02o_bench.err; echo "bench rc=$?"; tail -1 gpurun_out/r02o_bench.json | cut -c1-300
