#!/bin/bash
# Probe: warp-ring kernel vs the kernels it replaces on unaligned rows.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_softmax.py -q -x -k "warp_rings" > gpurun_out/ring_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/ring_tests.log
: > gpurun_out/ring_ab.jsonl
COLS="129,161,193,197,201,229,257,321,385,449,513,577,641,769,897,1001,1025,1281,1537,2047,2049,2561,3001,4097,5001,6145,8191,9215" \
MODES="QK_SM_RING=0;QK_SM_RING=1;QK_SM_RING=1,QK_SM_RING_NB=3" REPS=3 \
timeout 1500 python scripts/ring_ab.py >> gpurun_out/ring_ab.jsonl 2> gpurun_out/ring_err.log
COLS="10001,12001,14001,16387,20001" MODES="QK_SM_RING=0;QK_SM_RING=1;QK_SM_RING=1,QK_SM_RING_NB=3" REPS=3 \
timeout 1500 python scripts/ring_ab.py >> gpurun_out/ring_ab.jsonl 2>> gpurun_out/ring_err.log
