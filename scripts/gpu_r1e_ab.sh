# A/B on one box: old (popc + CUB scans), rank (two-launch bitmap rank), new (rank + fused count/scan); GPU suite on new
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1f_tests.log 2>&1; echo tests rc $?; tail -2 gpurun_out/r1f_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1f_smoke.log 2>&1; echo smoke rc $?; tail -1 gpurun_out/r1f_smoke.log
for rep in 1 2; do for cfg in mag synth_1b; do for v in old rank new; do
  if [ $v = new ]; then unset GSB_SO; else export GSB_SO=exp/$v.so; fi
  timeout 300 python bench.py --no-cpu-baseline --config $cfg --steps 400 > gpurun_out/r1f_${cfg}_${v}_$rep.log 2>&1
  tail -1 gpurun_out/r1f_${cfg}_${v}_$rep.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', '$v', round(d['value']), round(d['ms_per_step'],4), d['phase_ms_alone'], d['e2e']['value'])"
done; done; done
unset GSB_SO
CMD="python bench.py --no-cpu-baseline --steps 10 --warmup 3 --profile-steps 2"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:'gsb::|cub::' -s 300 -c 300 --csv --log-file gpurun_out/r1f_launches.csv $CMD > gpurun_out/r1f_ncu_launch.log 2>&1; echo launches rc $?
