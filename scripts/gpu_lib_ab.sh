#!/bin/bash
# Same-box A/B of two builds of libquake_b200.so on the cfg5 headline (back-to-back avg launch).
# usage: scripts/gpu_lib_ab.sh <B .so path> [rounds]
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
B=$1; N=${2:-4}
for i in $(seq 1 $N); do
  for v in A B; do
    if [ $v = A ]; then unset QK_LIB_PATH; else export QK_LIB_PATH=$B; fi
    timeout 300 python bench.py --no-extras --e2e-steps 1 --steps 40 2>&1 | python -c "import json,sys
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); r=d['roofline']; print('$v', round(r['avg_launch_us'],1), round(r['isolated_launch_us']['mean'],1), round(r['frac'],4))"
  done
done
unset QK_LIB_PATH
