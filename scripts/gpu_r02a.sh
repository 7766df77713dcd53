#!/bin/bash
# round 2 first check: GPU tests, C2 bench line, C3 anchor line at N=1, reference arm
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r02a_pytest.txt 2>&1
echo "pytest rc $?" >> gpurun_out/r02a_pytest.txt
timeout 600 python bench.py > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err
echo "bench rc $?" >> gpurun_out/r02a_bench.err
timeout 600 python bench.py --workload c3 --steps 5 > gpurun_out/r02a_c3.json 2> gpurun_out/r02a_c3.err
echo "c3 rc $?" >> gpurun_out/r02a_c3.err
timeout 600 python bench.py --impl reference --steps 5 > gpurun_out/r02a_ref.json 2> gpurun_out/r02a_ref.err
echo done
