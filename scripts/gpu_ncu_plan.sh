#!/bin/bash
# Tuning (not product): full ncu capture of one cfg5 softmax launch under a plan override.
#   scripts/gpu_ncu_plan.sh '<json env>' <kernel regex> <tag>
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
CMD="python scripts/sweep_softmax.py cfg5_softmax_vocab [$1]"
timeout 300 $CMD > gpurun_out/plain_$3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$2" -s 3 -c 1 -o gpurun_out/prof_$3 -f $CMD > gpurun_out/ncu_$3.log 2>&1
echo "ncu exit $?" >> gpurun_out/ncu_$3.log
python scripts/ncu_summary.py gpurun_out/prof_$3.ncu-rep gpurun_out/ncu_$3_summary "$3" > /dev/null 2>&1
python scripts/ncu_hot_sass.py gpurun_out/prof_$3.ncu-rep gpurun_out/ncu_$3_sass.txt 80
ncu -i gpurun_out/prof_$3.ncu-rep --page details --csv > gpurun_out/ncu_$3_details.csv 2>&1
rm -f gpurun_out/prof_$3.ncu-rep
ls -la gpurun_out
