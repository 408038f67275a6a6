# A/B round 2: default (agg 5 blocks/SM, one wave) vs 2 / 3 waves vs fill one wave; then the GPU suite
mkdir -p gpurun_out
for cfg in mag synth_1b; do for v in def w1 w2 w3 def; do
  if [ $v = def ]; then unset GSB_SO; else export GSB_SO=exp/$v.so; fi
  timeout 300 python bench.py --no-cpu-baseline --config $cfg --steps 300 > gpurun_out/ab2_${cfg}_$v.log 2>&1
  tail -1 gpurun_out/ab2_${cfg}_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['kernels']; print('$cfg', '$v', round(d['value']), round(d['ms_per_step'],4), round(k['rgcn_agg_l0']['us_per_step'],1), round(k['rgcn_agg_l1']['us_per_step'],1), round(k['sample_fill']['us_per_step'],1))"
done; done
unset GSB_SO
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/ab2_tests.log 2>&1; echo tests rc $?; tail -2 gpurun_out/ab2_tests.log
