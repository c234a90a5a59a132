#!/bin/bash
# Probe helper (not product): link each ab_objs/<name>.o (an alternative
# elementwise.o) with the other objects of the current build into
# /tmp/ab/libquake_b200_<name>.so, for QK_LIB_PATH A/B runs on the GPU box.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p /tmp/ab
B=paper_2412_00408_b200/build
for o in ab_objs/*.o; do
  n=$(basename "$o" .o)
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static \
    -o /tmp/ab/libquake_b200_$n.so "$o" $B/softmax.o $B/softmax_k_*.o $B/lab.o $B/host_api.o -lpthread
done
ls /tmp/ab
