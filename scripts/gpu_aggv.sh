# agg_l0 variants by build flags: usage bash scripts/gpu_aggv.sh TAG "FLAGS1" "FLAGS2" ...
T=$1; shift
for fl in "$@"; do
  GSB_NVCC_EXTRA="$fl" python -c "from paper_2406_06022_b200 import build; build.build(force=True)" > gpurun_out/${T}_build.log 2>&1
  for f in bf16 f32; do
    timeout 300 python bench.py --steps 300 --no-cpu-baseline --feat-dtype $f > gpurun_out/${T}_b.log 2>&1
    python3 -c "
import json; l=json.loads(open('gpurun_out/${T}_b.log').read().strip().splitlines()[-1]); r=l['roofline_kernels'].get('rgcn_agg_l0',{}); print('$fl', '$f', round(l['ms_per_step'],4), {k:round(v['us_per_step'],1) for k,v in l['kernels'].items() if 'agg' in k}, round(r.get('frac',0),3))"
  done
done
