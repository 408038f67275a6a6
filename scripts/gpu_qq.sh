for v in q3 q4 q3 q4; do
  cp scripts/libgsb_$v.bin paper_2406_06022_b200/libgsb.so
  for e in GSB_AGG_HALF=4; do
    env $e timeout 300 python bench.py --steps 300 --no-cpu-baseline > gpurun_out/qq_b.log 2>&1
    python3 -c "
import json; l=json.loads(open('gpurun_out/qq_b.log').read().strip().splitlines()[-1]); r=l['roofline_gather_aggregation'] or {}; print('$v', round(l['ms_per_step'],4), {k: round(v,4) for k,v in l['phase_ms_alone'].items()}, {k:round(v['us_per_step'],1) for k,v in l['kernels'].items() if 'agg' in k}, round(r.get('frac',0),3))"
  done
done
