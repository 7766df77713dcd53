#!/bin/bash
# session-4 final evidence: full GPU suite, smoke, default bench, reference arm,
# C3 line at N=1, the N=2 C3 path with two ranks sharing the GPU (gloo)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/s4z_pytest.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s4z_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4z_smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/s4z_smoke.txt
timeout 900 python bench.py > gpurun_out/s4z_bench.json 2> gpurun_out/s4z_bench.err; echo "bench rc=$?"; tail -1 gpurun_out/s4z_bench.json | cut -c1-160
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/s4z_ref.json 2> gpurun_out/s4z_ref.err; echo "ref rc=$?"; tail -1 gpurun_out/s4z_ref.json | cut -c1-160
timeout 600 python bench.py --workload c3 --steps 5 --no-cpu --no-sweep > gpurun_out/s4z_c3.json 2> gpurun_out/s4z_c3.err; echo "c3 rc=$?"; tail -1 gpurun_out/s4z_c3.json | cut -c1-160
FB_BENCH_BACKEND=gloo timeout 600 python bench.py --gpus 2 --workload c3 --steps 3 > gpurun_out/s4z_c3_2rank.json 2> gpurun_out/s4z_c3_2rank.err; echo "2rank rc=$?"; tail -1 gpurun_out/s4z_c3_2rank.json | cut -c1-160
