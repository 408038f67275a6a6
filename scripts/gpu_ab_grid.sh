# A/B of aggregation / sampling grid sizing (exp/*.so built with -D flags; GSB_SO selects)
mkdir -p gpurun_out
for cfg in mag synth_1b; do for v in v0 v1 v2 v3 v6 v4 v5 v0; do
  GSB_SO=exp/$v.so timeout 300 python bench.py --no-cpu-baseline --config $cfg --steps 300 > gpurun_out/ab_${cfg}_$v.log 2>&1
  tail -1 gpurun_out/ab_${cfg}_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$cfg', '$v', round(d['value']), round(d['ms_per_step'],4), d['phase_ms_alone'], round(k['rgcn_agg_l0']['us_per_step'],1), round(k['sample_fill']['us_per_step'],1))"
done; done
