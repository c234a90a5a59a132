#!/bin/bash
# Probe: rows per job / ring depth sweep of the warp-ring kernel.
# (run at commit acca6c1, the in-place + bulk-store form of the rings)
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
: > gpurun_out/ring_rj.jsonl
run() {  # cols, list of rj
  local c=$1; shift
  local modes=""
  for rj in "$@"; do
    for regs in 1 0; do
      for nb in 3 4; do
        modes="$modes;QK_SM_RING=1,QK_SM_RING_REGS=$regs,QK_SM_RING_RJ=$rj,QK_SM_RING_NB=$nb"
      done
    done
  done
  COLS=$c MODES="$modes" REPS=2 ITERS=6 timeout 300 python scripts/ring_ab.py >> gpurun_out/ring_rj.jsonl 2>> gpurun_out/ring_err.log
}
run 63 16 32 48 64
run 127 8 16 24 32 48
run 197 4 8 12 16 24
run 257 2 4 6 8 12 16
run 385 2 3 4 6 8
run 513 1 2 3 4 6
run 769 1 2 3 4
run 1001 1 2 3
run 1281 1 2
run 1537 1 2
run 2047 1
