#!/bin/bash
# Probe: warp-ring kernel, PDL trigger placement (entry vs after the last job).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
COLS="197,257,513,1001,1537,2049,4097,8191" MODES=";QK_SM_RING_LATE=1" REPS=3 \
timeout 1500 python scripts/ring_ab.py > gpurun_out/ring_late.jsonl 2> gpurun_out/ring_err.log
