# bulk-copy ring aggregation (agg_bulk_kernel, GSB_AGG=bulk): parity + bench A/B
T=$1
python -c "from paper_2406_06022_b200 import build; build.build()" > gpurun_out/${T}_build.log 2>&1; echo build rc $?
GSB_AGG=bulk timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_partition_sim.py -x -q > gpurun_out/${T}_tests.log 2>&1; echo tests rc $?; tail -5 gpurun_out/${T}_tests.log
summ() { python3 -c "
import json,sys; l=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=l['roofline']; print(sys.argv[2], round(l['ms_per_step'],4), l['phase_ms_alone'], r['kernel'], round(r['frac'],3), {k:round(v['us_per_step'],1) for k,v in l['kernels'].items() if 'agg' in k or 'gather' in k})" $1 "$2"; }
for e in "GSB_AGG=warp" "GSB_AGG=bulk" "GSB_AGGX=0"; do
  env $e timeout 300 python bench.py --steps 300 --no-cpu-baseline > gpurun_out/${T}_b_$e.log 2>&1; summ gpurun_out/${T}_b_$e.log "$e bf16"
  env $e timeout 300 python bench.py --steps 300 --no-cpu-baseline --feat-dtype f32 > gpurun_out/${T}_f_$e.log 2>&1; summ gpurun_out/${T}_f_$e.log "$e f32"
done
