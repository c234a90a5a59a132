#!/bin/bash
# Probe: ncu --set full of the warp-ring kernel at a few row lengths, with per-instruction counts.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
cap() {  # cols tag env...
  local cols=$1 tag=$2; shift 2
  env "$@" COLS=$cols MODES="" REPS=1 ITERS=2 TOTAL=${TOTAL:-67108864} timeout 300 ncu --set full --clock-control none --import-source on \
    -k regex:"softmax_wring" -s 2 -c 1 -o /tmp/ring_$tag -f python scripts/ring_ab.py > gpurun_out/ncu_ring_$tag.log 2>&1
  python scripts/ncu_summary.py /tmp/ring_$tag.ncu-rep gpurun_out/ncu_ring_$tag "$tag" > /dev/null 2>&1
  python scripts/ncu_inst_sass.py /tmp/ring_$tag.ncu-rep gpurun_out/ncu_ring_${tag}_inst.txt > /dev/null 2>&1
}
cap ${COLS1:-513} r513
cap ${COLS2:-77} r77
