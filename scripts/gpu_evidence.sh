#!/bin/bash
# Round evidence: smoke, GPU tests, bench (both arms, torchrun path), ncu
# launch list of the bench command, full ncu captures of the top kernels.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.csv 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 2400 python -m pytest tests -m gpu -q --timeout 900 -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/bench.log
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.log 2>&1; echo "ref exit $?" >> gpurun_out/bench_ref.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --steps 10 --warmup 3 --no-extras > gpurun_out/bench_torchrun.log 2>&1; echo "torchrun exit $?" >> gpurun_out/bench_torchrun.log
CMD="python bench.py --steps 3 --warmup 3 --no-extras --e2e-steps 1"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:softmax_pipe -s 3 -c 1 -o /tmp/prof_softmax_pipe -f $CMD > gpurun_out/ncu_full.log 2>&1
echo "ncu pipe exit $?" >> gpurun_out/ncu_full.log
CMD2="python scripts/kernel_probe.py"
timeout 300 $CMD2 > gpurun_out/kernel_probe.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:"ew_vec_kernel|softmax_subwarp" -c 6 -o /tmp/prof_ew -f $CMD2 > gpurun_out/ncu_ew.log 2>&1
echo "ncu ew exit $?" >> gpurun_out/ncu_ew.log
# summaries only (the full reports would exceed gpurun's 64 MiB copy-back)
python scripts/ncu_summary.py /tmp/prof_ew.ncu-rep gpurun_out/ncu_ew_summary "elementwise + warp softmax" > /dev/null 2>&1
python scripts/ncu_summary.py /tmp/prof_softmax_pipe.ncu-rep gpurun_out/ncu_pipe_summary "softmax_pipe cfg5" > /dev/null 2>&1
python scripts/ncu_hot_sass.py /tmp/prof_softmax_pipe.ncu-rep gpurun_out/ncu_pipe_sass.txt 80 > /dev/null 2>&1
ncu -i /tmp/prof_softmax_pipe.ncu-rep --page details --csv > gpurun_out/ncu_pipe_details.csv 2>&1
du -sh gpurun_out
# the 2-way split on one GPU through torchrun (correctness: fingerprints add up)
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 2 --steps 10 --warmup 3 --no-extras > gpurun_out/bench_torchrun2.log 2>&1; echo "torchrun2 exit $?" >> gpurun_out/bench_torchrun2.log
python scripts/launch_summary.py gpurun_out/launches.csv gpurun_out/launches_summary.json "$CMD" > /dev/null 2>&1
# softmax by row length with the final planner, and the warp-ring kernel under ncu
COLS="4,7,16,31,32,47,64,77,127,128,161,197,256,257,512,513,577,1001,1024,1025,2047,2049,4096,4097,8191,16384,16387,50000,50257,128256,151936,151937,202048,256000,262144" \
  timeout 900 python scripts/softmax_shape_sweep.py > gpurun_out/shape_sweep.jsonl 2> gpurun_out/shape_sweep.err
for c in 513 2049 4097; do
  COLS=$c MODES="" REPS=1 ITERS=2 TOTAL=268435456 timeout 300 ncu --set full --clock-control none --import-source on \
    -k regex:softmax_wring -s 2 -c 1 -o /tmp/ring_$c -f python scripts/ring_ab.py > gpurun_out/ncu_ring_$c.log 2>&1
  python scripts/ncu_summary.py /tmp/ring_$c.ncu-rep gpurun_out/ncu_ring_$c "warp-ring softmax, $c cols, QuAKE2" > /dev/null 2>&1
done
