#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_softmax.py -m gpu -q --timeout 400 -rf -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
QK_SM_CLUSTER=14 QK_SM_KC=15 QK_SM_THREADS=160 timeout 600 python -m pytest tests/test_gpu_softmax.py -m gpu -q --timeout 400 -rf -x -k "cfg5 or 128256 or 300000" > gpurun_out/pytest_gpu_forced.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_forced.log
timeout 400 python scripts/sweep_softmax.py > gpurun_out/sweep.log 2>&1; echo "sweep exit $?" >> gpurun_out/sweep.log
