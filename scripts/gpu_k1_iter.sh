#!/bin/bash
# K1 iteration: parity tests touching the refresh kernel, then timing.
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python scripts/exp_k1_diag.py 16 8
timeout 300 python scripts/exp_k1_diag.py 8 8
timeout 300 python scripts/trace_k1_graph.py 16 18 2>&1 | tail -2
