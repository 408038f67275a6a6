. scripts/summ.sh
for v in a b4 b5 b6; do
  for cfg in "mag" "mag --feat-dtype bf16" "synth_1b"; do
    GSB_SO=exp/libgsb_$v.so timeout 200 python bench.py --no-cpu-baseline --steps 200 --config $cfg > gpurun_out/b43.log 2>/dev/null
    python - "$v $cfg" <<'PY'
import json,sys
l=json.loads(open('gpurun_out/b43.log').read().strip().splitlines()[-1])
print(sys.argv[1], round(l['value']), 'agg_l0', round(l['kernels']['rgcn_agg_l0']['us_per_step'],1), 'agg_l1', round(l['kernels']['rgcn_agg_l1']['us_per_step'],1), 'roof', round(l['roofline']['frac'],3), l['roofline']['kernel'])
PY
  done
done
