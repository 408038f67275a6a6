# A/B on one box: {old .so, cur .so} x {GSB_PRIO=1 (compute graph on a high-priority stream), GSB_PRIO=0}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1i_tests.log 2>&1; echo tests rc $?; tail -2 gpurun_out/r1i_tests.log
for rep in 1 2; do for cfg in mag synth_1b; do for v in old cur; do for pr in 1 0; do
  if [ $v = cur ]; then unset GSB_SO; else export GSB_SO=exp/$v.so; fi
  GSB_PRIO=$pr timeout 300 python bench.py --no-cpu-baseline --config $cfg --steps 400 > gpurun_out/r1i_${cfg}_${v}_p${pr}_$rep.log 2>&1
  tail -1 gpurun_out/r1i_${cfg}_${v}_p${pr}_$rep.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', '$v', 'prio$pr', round(d['value']), round(d['ms_per_step'],4), d['phase_ms_alone'], round(d['e2e']['value']))"
done; done; done; done
unset GSB_SO
