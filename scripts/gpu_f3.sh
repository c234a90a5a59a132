#!/bin/bash
# §8(f3): GPU lab parity + acceptance tests, then the lab report.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_lab.py -m gpu -q --timeout 900 -rf > gpurun_out/pytest_f3.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_f3.log
timeout 900 python -m paper_2412_00408_b200.lab gpurun_out/lab_report.jsonl > gpurun_out/lab_report.log 2>&1; echo "exit $?" >> gpurun_out/lab_report.log
