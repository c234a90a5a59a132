#!/bin/bash
# Probe: elementwise logistic / GELU after the per-float4 division guard.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_elementwise.py -q -x > gpurun_out/ew_tests.log 2>&1
echo "tests exit $?" >> gpurun_out/ew_tests.log
: > gpurun_out/ew_inst.txt
for op in gelu logistic; do for k in 1 2; do
  timeout 200 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,sm__inst_issued.avg.pct_of_peak_sustained_active --clock-control none -k regex:ew_vec_kernel -s 2 -c 1 --csv \
    python scripts/ew_one.py $op $k 2>/dev/null | grep "ew_vec_kernel" | awk -F'","' -v o=$op -v k=$k '{print o, k, $(NF-2), $NF}' >> gpurun_out/ew_inst.txt
done; done
timeout 600 python bench.py --steps 10 --warmup 3 --e2e-steps 1 > gpurun_out/ew_bench.log 2>&1
