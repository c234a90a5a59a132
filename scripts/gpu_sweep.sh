#!/bin/bash
# Tuning run (not product): softmax parity under an env override, then a plan sweep.
#   scripts/gpu_sweep.sh '<env for the parity run>' '<json list of sweep envs>'
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
env $1 timeout 900 python -m pytest tests/test_gpu_softmax.py -m gpu -q --timeout 400 -rf -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python scripts/sweep_softmax.py "${3:-cfg5_softmax_vocab}" "$2" > gpurun_out/sweep.log 2>&1; echo "sweep exit $?" >> gpurun_out/sweep.log
