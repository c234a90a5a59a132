#!/bin/bash
# Probe: 16-warp agents for the warp rings at 12K-28K unaligned columns.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_softmax.py -q -x -k "warp_rings" > gpurun_out/ring_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/ring_tests.log
COLS="9215,12001,14001,16387,18001,20001,22001,24001,27001" \
MODES="QK_SM_RING=0;QK_SM_RING_MAX=30000,QK_SM_RING_AW=8;QK_SM_RING_MAX=30000,QK_SM_RING_AW=16;QK_SM_RING_MAX=30000" REPS=3 \
timeout 1500 python scripts/ring_ab.py > gpurun_out/ring_aw16.jsonl 2> gpurun_out/ring_err.log
