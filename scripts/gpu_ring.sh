#!/bin/bash
# Probe (not product): the warp-ring kernel against the other kernels for rows of
# cols % 4 != 0, interleaved in one process per row length (scripts/ring_ab.py).
#   QK_SM_RING=0  the planner without the rings (row spans up to 192 columns, else the
#                 scalar-lane cluster pipeline)
#   ""            the default planner (rings for 33-28000 unaligned columns)
#   QK_SM_RING_NB / QK_SM_RING_AW / QK_SM_RING_RJ / QK_SM_RING_REGS force the ring depth,
#                 warps per agent, rows per job, and the three-sweep form below 1025 columns
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_softmax.py -q -x -k "warp_rings" > gpurun_out/ring_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/ring_tests.log
COLS=${COLS:-"33,77,129,177,197,257,385,513,769,1001,1537,2049,3001,4097,8191,9215,12001,14001,16387,20001,27001"} \
MODES=${MODES:-"QK_SM_RING=0;;QK_SM_RING_NB=2;QK_SM_RING_NB=3"} REPS=3 \
timeout 1500 python scripts/ring_ab.py > gpurun_out/ring_ab.jsonl 2> gpurun_out/ring_err.log
