# quick A/B of knobs on the default bench.  usage: bash scripts/gpu_quick.sh TAG "ENV1" "ENV2" ...
T=$1; shift
python -c "from paper_2406_06022_b200 import build; build.build()" > gpurun_out/${T}_build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gemm.py -x -q -k "nc_ or step or splitk or gcn" > gpurun_out/${T}_tests.log 2>&1; echo tests rc $?; tail -1 gpurun_out/${T}_tests.log
i=0
for e in "$@"; do
  i=$((i+1))
  env $e timeout 300 python bench.py --steps 300 --no-cpu-baseline > gpurun_out/${T}_b$i.log 2>&1
  python3 -c "
import json; l=json.loads(open('gpurun_out/${T}_b$i.log').read().strip().splitlines()[-1]); print('$e', round(l['ms_per_step'],4), l['phase_ms_alone'], {k:round(v['us_per_step'],1) for k,v in l['kernels'].items() if 'gemm' in k or 'nc_' in k or 'scatter' in k or 'relu' in k or 'tcsr' in k})"
done
