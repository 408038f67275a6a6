timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | grep -E "Error|error|assert|FAILED|passed|failed|mismatch" | head -10
for rw in 1 2 4; do
  GSB_AGG_RW=$rw timeout 300 python bench.py --no-cpu-baseline --steps 200 > gpurun_out/agg7_$rw.log 2>&1; echo rc $?
  python - <<PY
import json; d=json.loads(open("gpurun_out/agg7_$rw.log").read().strip().splitlines()[-1])
print("rw$rw", d["value"], d["ms_per_step"], {k:v["us_per_step"] for k,v in d["kernels"].items() if "agg" in k})
PY
done
