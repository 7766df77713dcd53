#!/bin/bash
# session-4 fresh-container evidence: full GPU suite, smoke, default bench, reference arm,
# C3 line at N=1, bench launch list under ncu
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/r02s4_pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02s4_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02s4_smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02s4_smoke.txt
timeout 900 python bench.py > gpurun_out/r02s4_bench.json 2> gpurun_out/r02s4_bench.err; echo "bench rc=$?"; tail -1 gpurun_out/r02s4_bench.json | cut -c1-200
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02s4_ref.json 2> gpurun_out/r02s4_ref.err; echo "ref rc=$?"; tail -1 gpurun_out/r02s4_ref.json | cut -c1-200
timeout 600 python bench.py --workload c3 --steps 5 --no-cpu --no-sweep > gpurun_out/r02s4_c3.json 2> gpurun_out/r02s4_c3.err; echo "c3 rc=$?"; tail -1 gpurun_out/r02s4_c3.json | cut -c1-200

