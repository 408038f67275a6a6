for neg in joint uniform local_joint in_batch; do
  timeout 600 python bench.py --no-cpu-baseline --config amazon_lp --steps 50 --warmup 5 --profile-steps 3 --neg $neg > gpurun_out/neg2_$neg.log 2>&1; echo rc $?
  python - <<PY
import json; d=json.loads(open("gpurun_out/neg2_$neg.log").read().strip().splitlines()[-1])
print("$neg", d["value"], d["ms_per_step"], d["config"]["workload"], sorted(((round(v["us_per_step"]),k) for k,v in d["kernels"].items()), reverse=True)[:5])
PY
done
timeout 600 python bench.py --no-cpu-baseline --config amazon_lp --steps 50 --warmup 5 --profile-steps 3 --score dot > gpurun_out/neg2_dot.log 2>&1; echo rc $?
python -c "import json; d=json.loads(open('gpurun_out/neg2_dot.log').read().strip().splitlines()[-1]); print('dot', d['value'], d['ms_per_step'])"
