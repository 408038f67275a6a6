# quarter-warp-per-row layer-0 aggregation (GSB_AGG_HALF=4) vs the size-selected default
python -c "from paper_2406_06022_b200 import build; build.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "optin or full_scale or mag_bf16" > gpurun_out/qt_tests.log 2>&1; echo tests rc $?; tail -1 gpurun_out/qt_tests.log
for a in "" "--config amazon_lp" "--config synth_1b"; do
  for e in X=1 GSB_AGG_HALF=4 X=1 GSB_AGG_HALF=4; do
    env $e timeout 300 python bench.py --steps 300 --no-cpu-baseline $a > gpurun_out/qt_b.log 2>&1
    python3 -c "
import json; l=json.loads(open('gpurun_out/qt_b.log').read().strip().splitlines()[-1]); r=l['roofline_gather_aggregation'] or {}; print('$a', '$e', round(l['ms_per_step'],4), {k: round(v,4) for k,v in l['phase_ms_alone'].items()}, {k:round(v['us_per_step'],1) for k,v in l['kernels'].items() if 'agg' in k}, round(r.get('frac',0),3))"
  done
done
