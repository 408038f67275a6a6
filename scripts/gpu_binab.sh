# A/B of prebuilt libgsb variants (scripts/libgsb_<v>.bin, built here with GSB_NVCC_EXTRA):
# usage bash scripts/gpu_binab.sh TAG FILTER "CONFIG_ARGS" v1 v2 ...   (mag bench, 300 steps)
T=$1; F=$2; A=$3; shift 3
for v in "$@"; do
  cp scripts/libgsb_$v.bin paper_2406_06022_b200/libgsb.so
  timeout 300 python bench.py --steps 300 --no-cpu-baseline $A > gpurun_out/${T}_b.log 2>&1
  python3 -c "
import json; l=json.loads(open('gpurun_out/${T}_b.log').read().strip().splitlines()[-1]); print('$v', round(l['ms_per_step'],4), {k: round(v,4) for k,v in l['phase_ms_alone'].items()}, {k:round(v['us_per_step'],1) for k,v in l['kernels'].items() if '$F' in k})"
done
