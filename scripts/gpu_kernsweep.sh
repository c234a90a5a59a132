#!/bin/bash
# Tuning (not product): plan sweep per kernel choice for one workload.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
: > gpurun_out/kernsweep.log
for k in $2; do
  echo "== kernel $k" >> gpurun_out/kernsweep.log
  SWEEP_KERNEL=$k timeout 300 python scripts/sweep_softmax.py "$3" "$1" >> gpurun_out/kernsweep.log 2>&1
done
