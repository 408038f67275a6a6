# weight images A/B + correctness.  usage: bash scripts/gpu_wimg.sh TAG
T=${1:-wi}
python -c "from paper_2406_06022_b200 import build; build.build()" > gpurun_out/${T}_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gemm.py tests/test_gpu_lp.py tests/test_gpu_negatives.py tests/test_gpu_partition_sim.py -x -q > gpurun_out/${T}_tests.log 2>&1; echo tests rc $?; tail -2 gpurun_out/${T}_tests.log
. scripts/summ.sh
for w in img noimg; do
  if [ $w = noimg ]; then export GSB_NO_WIMG=1; else unset GSB_NO_WIMG; fi
  timeout 300 python bench.py --steps 200 --no-cpu-baseline > gpurun_out/${T}_bench_$w.log 2>&1; echo bench $w rc $?
  summ gpurun_out/${T}_bench_$w.log | head -3
  python3 -c "
import json; l=json.loads(open('gpurun_out/${T}_bench_$w.log').read().strip().splitlines()[-1]); print(l['phase_ms_alone']); print({k:round(v['us_per_step'],1) for k,v in l['kernels'].items() if 'gemm' in k or 'nc_' in k or 'weight' in k})"
done
