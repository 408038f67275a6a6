# SIMT small-GEMM path (gemm_simt.cuh): micro A/B, parity, bench A/B
T=$1
python -c "from paper_2406_06022_b200 import build; build.build()" > gpurun_out/${T}_build.log 2>&1; echo build rc $?
for e in "GSB_SIMT=1" "GSB_SIMT=0"; do env $e SHAPES=1024x640x128,1024x128x352,1024x128x128 timeout 120 python scripts/gemm_micro.py 2>&1 | grep mode | sed "s/^/$e /" | cut -c1-120; done
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py tests/test_gpu_lp.py tests/test_gpu_inference.py -x -q > gpurun_out/${T}_tests.log 2>&1; echo tests rc $?; tail -3 gpurun_out/${T}_tests.log
for e in "GSB_SIMT=0" "GSB_SIMT=1" "GSB_SIMT=0" "GSB_SIMT=1"; do
  env $e timeout 300 python bench.py --steps 300 --no-cpu-baseline > gpurun_out/${T}_b.log 2>&1
  python3 -c "
import json; l=json.loads(open('gpurun_out/${T}_b.log').read().strip().splitlines()[-1]); print('$e', round(l['ms_per_step'],4), l['phase_ms_alone'], {k:round(v['us_per_step'],1) for k,v in l['kernels'].items() if 'gemm' in k or 'nc_' in k})"
done
