# input encoder with TMA-fed B operands: parity + MAG240M 1/16 bench A/B (GSB_ENC_TMA=0 = cp.async B)
T=$1
python -c "from paper_2406_06022_b200 import build; build.build()" > gpurun_out/${T}_build.log 2>&1; echo build rc $?
timeout 900 python -m pytest tests/test_gpu_encoder.py tests/test_gpu_parity.py -x -q > gpurun_out/${T}_tests.log 2>&1; echo tests rc $?; tail -3 gpurun_out/${T}_tests.log
for e in "GSB_ENC_TMA=0" "GSB_ENC_TMA=1" "GSB_ENC_TMA=0" "GSB_ENC_TMA=1"; do
  env $e timeout 600 python bench.py --config mag240m_1_16 --steps 200 --no-cpu-baseline > gpurun_out/${T}_b.log 2>&1
  python3 -c "
import json; l=json.loads(open('gpurun_out/${T}_b.log').read().strip().splitlines()[-1]); print('$e', round(l['ms_per_step'],4), l['phase_ms_alone'], {k:round(v['us_per_step'],1) for k,v in l['kernels'].items() if 'enc' in k})"
done
