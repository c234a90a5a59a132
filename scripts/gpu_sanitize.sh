#!/bin/bash
# compute-sanitizer over scripts/sanitize_probe.py (memcheck, racecheck, synccheck).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 300 python scripts/sanitize_probe.py > gpurun_out/sanitize_plain.log 2>&1; echo "exit $?" >> gpurun_out/sanitize_plain.log
for tool in memcheck racecheck synccheck; do
  timeout 1200 $CS --tool $tool --print-limit 20 python scripts/sanitize_probe.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "exit $?" >> gpurun_out/sanitize_$tool.log
done
