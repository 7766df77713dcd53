#!/bin/bash
# round 2: config-size oracle parity + the reference's verification / acceptance suites on the device
cd $GRAFT_REPO_ROOT
rm -f gpurun_out/config_parity.jsonl
timeout 1500 python -m pytest tests/test_config_parity.py tests/test_reference_suites.py -m gpu -q -rA --durations=30 > gpurun_out/r02b_pytest.txt 2>&1
echo "pytest rc $?" >> gpurun_out/r02b_pytest.txt
timeout 300 python bench.py --steps 20 --no-sweep --no-cpu > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err
