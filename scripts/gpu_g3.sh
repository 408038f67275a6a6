# TMA-everything GEMM (gemm_tma3.cuh): micro A/B, GEMM + step parity, bench A/B over env variants
# usage: bash scripts/gpu_g3.sh TAG "ENV1" "ENV2" ...
T=$1; shift
python -c "from paper_2406_06022_b200 import build; build.build()" > gpurun_out/${T}_build.log 2>&1; echo build rc $?
for g in tma2 tma3; do GSB_GEMM=$g timeout 120 python scripts/gemm_micro.py > gpurun_out/${T}_micro_$g.log 2>&1; echo micro $g rc $?; cat gpurun_out/${T}_micro_$g.log | grep mode; done
M=1024 GSB_GEMM_DBG=5120 timeout 60 python scripts/gemm_trace.py 2>&1 | grep epi
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py -x -q > gpurun_out/${T}_tests.log 2>&1; echo tests rc $?; tail -3 gpurun_out/${T}_tests.log
i=0
for e in "$@"; do
  i=$((i+1))
  env $e timeout 300 python bench.py --steps 300 --no-cpu-baseline > gpurun_out/${T}_b$i.log 2>&1
  python3 -c "
import json; l=json.loads(open('gpurun_out/${T}_b$i.log').read().strip().splitlines()[-1]); print('$e', round(l['ms_per_step'],4), l['phase_ms_alone'], {k:round(v['us_per_step'],1) for k,v in l['kernels'].items() if 'gemm' in k or 'nc_' in k})"
done
