#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/r02l_pytest.txt 2>&1; echo "pytest rc $?" >> gpurun_out/r02l_pytest.txt
tail -2 gpurun_out/r02l_pytest.txt
timeout 600 python bench.py --workload c3 --steps 5 > gpurun_out/r02l_c3.json 2> gpurun_out/r02l_c3.err; echo "c3 rc $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02l_ref.json 2> gpurun_out/r02l_ref.err; echo "ref rc $?"
