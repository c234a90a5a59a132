#!/bin/bash
# Full GPU tests, then bench under two environments (A/B), e.g. QK_PDL=1 vs QK_PDL=0.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
env $1 timeout 600 python bench.py > gpurun_out/bench_a.log 2>&1; echo "exit $?" >> gpurun_out/bench_a.log
env $2 timeout 600 python bench.py > gpurun_out/bench_b.log 2>&1; echo "exit $?" >> gpurun_out/bench_b.log
