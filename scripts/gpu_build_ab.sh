#!/bin/bash
# Same-box A/B of two builds of libquake_b200.so (QK_LIB_PATH = the B build) over softmax row
# lengths and the elementwise configs: one short process per measurement, alternating builds.
# usage: scripts/gpu_build_ab.sh <B .so path>
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
B=$1
: > gpurun_out/build_ab.jsonl
for c in ${COLS:-47 197 257 513 1001 1537 2049 4097 8191 12001 16387 50257 512 4096 16384 50000 128256 262144}; do
  for v in A B A B; do
    if [ $v = A ]; then unset QK_LIB_PATH; else export QK_LIB_PATH=$B; fi
    COLS=$c MODES="" REPS=2 ITERS=8 timeout 120 python scripts/ring_ab.py 2>/dev/null | sed "s/^{/{\"build\": \"$v\", /" >> gpurun_out/build_ab.jsonl
  done
done
unset QK_LIB_PATH
for v in A B A B; do
  if [ $v = A ]; then unset QK_LIB_PATH; else export QK_LIB_PATH=$B; fi
  timeout 600 python bench.py --steps 20 --warmup 5 --e2e-steps 1 2>/dev/null | grep '^{' | sed "s/^{/{\"build\": \"$v\", /" >> gpurun_out/build_ab_bench.jsonl
done
