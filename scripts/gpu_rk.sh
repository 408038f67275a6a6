T=$1
python -c "from paper_2406_06022_b200 import build; build.build()" > gpurun_out/${T}_build.log 2>&1; echo build rc $?
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${T}_tests.log 2>&1; echo tests rc $?; tail -2 gpurun_out/${T}_tests.log
for e in GSB_RANK_FUSED=0 GSB_RANK_FUSED=1 GSB_RANK_FUSED=0 GSB_RANK_FUSED=1; do
  env $e timeout 300 python bench.py --steps 300 --no-cpu-baseline > gpurun_out/${T}_b.log 2>&1
  python3 -c "
import json; l=json.loads(open('gpurun_out/${T}_b.log').read().strip().splitlines()[-1]); print('$e', round(l['ms_per_step'],4), l['phase_ms_alone'], {k:round(v['us_per_step'],1) for k,v in l['kernels'].items() if 'rank' in k or 'meta' in k})"
done
