# half-warp-per-row layer-0 aggregation: parity + A/B against the warp kernel (GSB_AGG_HALF=0 warp,
# unset = size-selected default, 2 = forced)
python -c "from paper_2406_06022_b200 import build; build.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/hf_tests.log 2>&1; echo tests rc $?; tail -1 gpurun_out/hf_tests.log
for a in "" "--config amazon_lp" "--feat-dtype f32"; do
  for e in ${ENVS:-GSB_AGG_HALF=0 GSB_AGG_HALF=1 GSB_AGG_HALF=0 GSB_AGG_HALF=1}; do
    env $e timeout 300 python bench.py --steps 300 --no-cpu-baseline $a > gpurun_out/hf_b.log 2>&1
    python3 -c "
import json; l=json.loads(open('gpurun_out/hf_b.log').read().strip().splitlines()[-1]); print('$a', '$e', round(l['ms_per_step'],4), {k: round(v,4) for k,v in l['phase_ms_alone'].items()}, {k:round(v['us_per_step'],1) for k,v in l['kernels'].items() if 'agg' in k}, l['roofline']['kernel'], round(l['roofline']['frac'],3))"
  done
done
