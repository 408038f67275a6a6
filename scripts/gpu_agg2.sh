# agg_l0 with row-level key prefetch: parity + bench (bf16 / f32) agg times
T=$1
python -c "from paper_2406_06022_b200 import build; build.build()" > gpurun_out/${T}_build.log 2>&1; echo build rc $?
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition_sim.py tests/test_gpu_fullscale.py tests/test_gpu_inference.py -x -q > gpurun_out/${T}_tests.log 2>&1; echo tests rc $?; tail -2 gpurun_out/${T}_tests.log
for f in bf16 f32 bf16 f32; do
  timeout 300 python bench.py --steps 300 --no-cpu-baseline --feat-dtype $f > gpurun_out/${T}_b.log 2>&1
  python3 -c "
import json; l=json.loads(open('gpurun_out/${T}_b.log').read().strip().splitlines()[-1]); r=[x for x in l.get('roofline_kernels',[]) if x.get('kernel')=='rgcn_agg_l0']; print('$f', round(l['ms_per_step'],4), l['phase_ms_alone'], {k:round(v['us_per_step'],1) for k,v in l['kernels'].items() if 'agg' in k}, [round(x['frac'],3) for x in r])"
done
