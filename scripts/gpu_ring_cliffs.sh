#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
C=""; for c in $(seq 2049 64 2753) $(seq 4545 96 5409) $(seq 9025 128 9921) $(seq 13057 256 15617) 18001 22001 26001 27999; do C="$C,$c"; done
COLS="${C#,}" MODES="" REPS=2 timeout 1500 python scripts/ring_ab.py > gpurun_out/ring_cliffs.jsonl 2> gpurun_out/ring_err.log
C=""; for c in $(seq 33 8 193) $(seq 193 24 1057); do [ $((c % 4)) -ne 0 ] && C="$C,$c"; done
COLS="${C#,}" MODES="" REPS=2 timeout 1500 python scripts/ring_ab.py >> gpurun_out/ring_cliffs.jsonl 2>> gpurun_out/ring_err.log
