#!/bin/bash
# Probe: lanes per row (G) x rows per job sweep of the register-form warp ring.
# (run at commit acca6c1: the QK_SM_RING_G knob it used was folded into the planner afterwards)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
: > gpurun_out/ring_g.jsonl
for c in ${COLS:-47 63 77 97 127 129 161 197 229 257 321 385 449 513 641}; do
  modes=""
  for g in 4 8 16 32; do
    need=$(( (c + g - 1) / g ))
    [ $need -gt 32 ] && continue
    [ $g -eq 4 ] && [ $need -gt 24 ] && continue
    per=$(( 32 / g ))
    for kb in 2048 4096 6144; do
      rj=$(( (kb + c*2) / (c*4) )); rj=$(( (rj + per - 1) / per * per ))
      modes="$modes;QK_SM_RING=1,QK_SM_RING_G=$g,QK_SM_RING_RJ=$rj,QK_SM_RING_NB=3"
    done
  done
  COLS=$c MODES="$modes" REPS=2 ITERS=6 timeout 300 python scripts/ring_ab.py >> gpurun_out/ring_g.jsonl 2>> gpurun_out/ring_err.log
done
