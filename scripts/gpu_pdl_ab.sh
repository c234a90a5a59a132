mkdir -p gpurun_out
for v in "QK_PDL=0" "QK_PDL=1 QK_PDL_LATE=0" "QK_PDL=1 QK_PDL_LATE=1" "QK_PDL=0" "QK_PDL=1 QK_PDL_LATE=0" "QK_PDL=1 QK_PDL_LATE=1"; do
  echo "== $v" >> gpurun_out/pdl_ab.log
  env $v timeout 300 python bench.py --steps 20 --warmup 3 --no-extras --e2e-steps 1 2>&1 | python -c "import json,sys
for l in sys.stdin:
  if l.startswith('{'):
    d=json.loads(l); r=d['roofline']; print(round(r['avg_launch_us'],1), r['isolated_launch_us'], round(r['frac'],4))
  else: print(l.rstrip())" >> gpurun_out/pdl_ab.log
done
