#!/bin/bash
# bf16 cached partial: new parity tests, full GPU suite, bench, K2 A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_partial_bf16.py -m gpu -q -rf > gpurun_out/r02d_pb16.txt 2>&1
echo "pb16 rc $?" >> gpurun_out/r02d_pb16.txt
timeout 1500 python -m pytest tests -m gpu -q -x -rf > gpurun_out/r02d_pytest.txt 2>&1
echo "pytest rc $?" >> gpurun_out/r02d_pytest.txt
timeout 300 python scripts/ab_k2_extb.py 16 8 4 > gpurun_out/r02d_ab_k2.txt 2>&1
timeout 600 python bench.py --no-sweep --no-cpu > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err
echo "bench rc $?" >> gpurun_out/r02d_bench.err
