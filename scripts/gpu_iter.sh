#!/bin/bash
# iteration: GPU parity tests, then A/B bench vs scripts/micro/libfb200_old.so
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
bash scripts/gpu_ab.sh
