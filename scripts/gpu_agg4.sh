timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
for v in 1 0; do
  for dt in bf16 f32; do
  GSB_AGG=$v timeout 300 python bench.py --no-cpu-baseline --steps 200 --feat-dtype $dt > gpurun_out/agg3_${dt}_v$v.log 2>&1; echo rc $?
  python - <<PY
import json; d=json.loads(open("gpurun_out/agg3_${dt}_v$v.log").read().strip().splitlines()[-1])
print("$dt v$v", d["value"], d["ms_per_step"], d["roofline_gather_aggregation"]["avg_launch_us"], d["roofline_gather_aggregation"]["frac"], {k:v["us_per_step"] for k,v in d["kernels"].items() if "agg" in k})
PY
  done
done
GSB_AGG=1 timeout 300 python bench.py --no-cpu-baseline --steps 200 --config synth_1b > gpurun_out/agg3_1b.log 2>&1; tail -c 300 gpurun_out/agg3_1b.log
CMD="python bench.py --no-cpu-baseline --steps 3 --warmup 3 --profile-steps 1 --no-graph"
GSB_AGG=1 timeout 300 $CMD > gpurun_out/agg3_plain.log 2>&1 && GSB_AGG=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:"agg" -s 4 -c 2 -o gpurun_out/agg3_v1 $CMD > gpurun_out/agg3_ncu.log 2>&1; echo rc $?
