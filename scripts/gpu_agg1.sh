set -x
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -5
for v in 1 0; do
  GSB_AGG=$v timeout 300 python bench.py --no-cpu-baseline --steps 200 > gpurun_out/agg_v$v.log 2>&1; echo rc $?
  python - <<PY
import json; d=json.loads(open("gpurun_out/agg_v$v.log").read().strip().splitlines()[-1])
print("v$v", d["value"], d["ms_per_step"], d["roofline"]["avg_launch_us"], d["roofline"]["frac"], {k:v["us_per_step"] for k,v in d["kernels"].items() if "agg" in k})
PY
  GSB_AGG=$v timeout 300 python bench.py --no-cpu-baseline --steps 200 --feat-dtype f32 > gpurun_out/agg_f32_v$v.log 2>&1; echo rc $?
  python - <<PY
import json; d=json.loads(open("gpurun_out/agg_f32_v$v.log").read().strip().splitlines()[-1])
print("f32 v$v", d["value"], d["ms_per_step"], d["roofline"]["avg_launch_us"], d["roofline"]["frac"], {k:v["us_per_step"] for k,v in d["kernels"].items() if "agg" in k})
PY
done
