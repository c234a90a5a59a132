#!/bin/bash
# §8(f2): ablation parity tests, then the GPU Table III and the kernel matrix.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ablation.py tests/test_gpu_softmax.py -m gpu -q --timeout 600 -rf -x > gpurun_out/pytest_f2.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_f2.log
timeout 600 python -m paper_2412_00408_b200.ablation --mode table3 > gpurun_out/ablation_table3.jsonl 2> gpurun_out/ablation_table3.err; echo "exit $?" >> gpurun_out/ablation_table3.err
timeout 600 python -m paper_2412_00408_b200.ablation --mode table3 --rows 4096 --cols 128256 --n 67108864 > gpurun_out/ablation_table3_large.jsonl 2>> gpurun_out/ablation_table3.err; echo "exit $?" >> gpurun_out/ablation_table3.err
timeout 600 python -m paper_2412_00408_b200.ablation --mode matrix --rows 16384 --cols 16384 --n 67108864 > gpurun_out/ablation_matrix.jsonl 2> gpurun_out/ablation_matrix.err; echo "exit $?" >> gpurun_out/ablation_matrix.err
