#!/bin/bash
# session-4 closing check of the final tree: full GPU suite and smoke
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -rf > gpurun_out/s4m_pytest.txt 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/s4m_pytest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s4m_smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/s4m_smoke.txt
