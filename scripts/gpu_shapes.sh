#!/bin/bash
# Tuning (not product): default plan vs alternatives over several row lengths.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
: > gpurun_out/shapes.log
for spec in "cfg5_softmax_vocab" "paper_softmax_16k" "shape:65536x2048" "shape:32768x4096" "shape:8192x50000" "shape:2048x300000" "shape:65536x1536"; do
  echo "== $spec" >> gpurun_out/shapes.log
  timeout 300 python scripts/sweep_softmax.py "$spec" "$1" >> gpurun_out/shapes.log 2>&1
done
