#!/bin/bash
# Probe: warp-ring kernel (direct stores) below 193 columns vs the row-span kernel.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
COLS="33,41,47,49,63,65,77,97,111,127,129,145,161,177,191" \
MODES=";QK_SM_RING=1;QK_SM_RING=1,QK_SM_RING_NB=2;QK_SM_RING=1,QK_SM_RING_NB=3" REPS=3 \
timeout 1500 python scripts/ring_ab.py > gpurun_out/ring_short.jsonl 2> gpurun_out/ring_err.log
