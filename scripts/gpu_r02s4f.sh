#!/bin/bash
# session-4: K2 defaults by grid size -- full GPU suite, A/B incl. defaults, bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/ab_k2_store.py 4 16 32 64 > gpurun_out/s4f_ab.txt 2>&1; echo "ab rc=$?"; grep -v "equal" gpurun_out/s4f_ab.txt | tail -20
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/s4f_pytest.txt 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/s4f_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4f_smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/s4f_smoke.txt
timeout 900 python bench.py > gpurun_out/s4f_bench.json 2> gpurun_out/s4f_bench.err; echo "bench rc=$?"; tail -1 gpurun_out/s4f_bench.json | cut -c1-200
