#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/r02j_pytest.txt 2>&1; echo "pytest rc $?" >> gpurun_out/r02j_pytest.txt
tail -2 gpurun_out/r02j_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r02j_bench.json 2> gpurun_out/r02j_bench.err; echo "bench rc $?"
