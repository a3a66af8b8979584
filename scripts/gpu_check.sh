#!/bin/bash
# GPU-box helper: run the GPU parity tests and record the environment.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/nvsmi.txt 2>&1
timeout ${PYTEST_TIMEOUT:-900} python -m pytest ${PYTEST_ARGS:-tests -m gpu -x -q} > gpurun_out/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
tail -60 gpurun_out/pytest_gpu.txt
