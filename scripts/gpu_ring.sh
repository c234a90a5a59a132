#!/bin/bash
# Probe: warp-ring kernel (direct stores): ring depth, job size, upper end of its range.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_softmax.py -q -x -k "warp_rings" > gpurun_out/ring_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/ring_tests.log
COLS="197,257,385,513,769,1001,1281,1537,2049,3001,4097,6145,8191,9215,10001,12001,14001,16387,20001" \
MODES="QK_SM_RING=0;QK_SM_RING_MAX=32000;QK_SM_RING_MAX=32000,QK_SM_RING_NB=2;QK_SM_RING_MAX=32000,QK_SM_RING_NB=3" REPS=3 \
timeout 1500 python scripts/ring_ab.py > gpurun_out/ring_direct2.jsonl 2> gpurun_out/ring_err.log
: > gpurun_out/ring_rj2.jsonl
for c in 197 257 513 1001; do
  modes=""
  for kb in 3072 4096 6144 8192 12288; do
    g=8; [ $c -gt 256 ] && g=16; [ $c -gt 512 ] && g=32; per=$(( 32 / g ))
    rj=$(( (kb + c*2) / (c*4) )); rj=$(( (rj + per - 1) / per * per ))
    modes="$modes;QK_SM_RING_RJ=$rj"
  done
  COLS=$c MODES="${modes#;}" REPS=3 timeout 300 python scripts/ring_ab.py >> gpurun_out/ring_rj2.jsonl 2>> gpurun_out/ring_err.log
done
