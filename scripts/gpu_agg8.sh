timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | grep -E "Error|error|assert|FAILED|passed|failed|mismatch" | head -10
for cfg in mag synth_1b mag240m_1_16; do
  timeout 300 python bench.py --no-cpu-baseline --steps 200 --config $cfg > gpurun_out/agg8_$cfg.log 2>&1; echo rc $?
  python - <<PY
import json; d=json.loads(open("gpurun_out/agg8_$cfg.log").read().strip().splitlines()[-1])
print("$cfg", d["value"], d["ms_per_step"], {k:v["us_per_step"] for k,v in d["kernels"].items() if "agg" in k})
PY
done
