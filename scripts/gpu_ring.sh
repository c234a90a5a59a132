#!/bin/bash
# Probe: after building without relocatable device code — bench line and the unaligned-row sweep.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c.log 2>&1; echo "bench exit $?" >> gpurun_out/bench_c.log
COLS="47,127,197,257,385,513,769,1001,1537,2049,3001,4097,8191,12001,16387,50257" MODES="" REPS=3 \
timeout 900 python scripts/ring_ab.py > gpurun_out/ring_c.jsonl 2> gpurun_out/ring_err.log
COLS="512,4096,16384,50000,128256,202048,262144" MODES="" REPS=3 \
timeout 900 python scripts/ring_ab.py >> gpurun_out/ring_c.jsonl 2>> gpurun_out/ring_err.log
