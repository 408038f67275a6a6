# A/B on one box: GSB_PRIO = 0 (default priorities), 1 (compute stream high), 2 (sample side stream high)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/r1j_tests.log 2>&1; echo tests rc $?; tail -2 gpurun_out/r1j_tests.log
for rep in 1 2; do for cfg in mag synth_1b; do for pr in 0 1 2; do
  GSB_PRIO=$pr timeout 300 python bench.py --no-cpu-baseline --config $cfg --steps 400 > gpurun_out/r1j_${cfg}_p${pr}_$rep.log 2>&1
  tail -1 gpurun_out/r1j_${cfg}_p${pr}_$rep.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', 'prio$pr', round(d['value']), round(d['ms_per_step'],4), d['phase_ms_alone'], round(d['e2e']['value']))"
done; done; done
timeout 600 python bench.py > gpurun_out/r1j_bench_default.log 2>&1; echo bench rc $?; tail -1 gpurun_out/r1j_bench_default.log | head -c 300; echo
