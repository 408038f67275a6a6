# quarter-warp layer-0 aggregation as the default: GPU suite + mag / amazon_lp / synth_1b / f32 benches
python -c "from paper_2406_06022_b200 import build; build.build()" > /dev/null 2>&1
timeout 700 python -m pytest tests -m gpu -q > gpurun_out/qd_tests.log 2>&1; echo tests rc $?; tail -1 gpurun_out/qd_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for a in "" "--config amazon_lp" "--config synth_1b" "--feat-dtype f32"; do
  for e in X=1 GSB_AGG_HALF=0; do
    env $e timeout 300 python bench.py --steps 300 --no-cpu-baseline $a > gpurun_out/qd_b.log 2>&1
    python3 -c "
import json; l=json.loads(open('gpurun_out/qd_b.log').read().strip().splitlines()[-1]); r=l['roofline_gather_aggregation'] or {}; print('$a', '$e', round(l['ms_per_step'],4), round(l['e2e']['value']/1e6,3), {k: round(v,4) for k,v in l['phase_ms_alone'].items()}, {k:round(v['us_per_step'],1) for k,v in l['kernels'].items() if 'agg' in k}, round(r.get('frac',0),3))"
  done
done
