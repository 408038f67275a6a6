# LP bench A/B over env variants: usage bash scripts/gpu_lpq.sh TAG "ENV" ...
T=$1; shift
python -c "from paper_2406_06022_b200 import build; build.build()" > gpurun_out/${T}_build.log 2>&1
for e in "$@"; do
  env $e timeout 600 python bench.py --config amazon_lp --steps 100 --no-cpu-baseline > gpurun_out/${T}_b.log 2>&1
  python3 -c "
import json; l=json.loads(open('gpurun_out/${T}_b.log').read().strip().splitlines()[-1]); print('$e', round(l['ms_per_step'],4), l['phase_ms_alone'], {k:round(v['us_per_step'],1) for k,v in l['kernels'].items() if 'agg' in k or 'gemm_fwd_l0' in k})"
done
