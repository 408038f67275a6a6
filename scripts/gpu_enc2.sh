# encoder decoupled A/B rings: parity + MAG240M 1/16 bench A/B against the previous binary
T=$1
cp scripts/libgsb_${FIRST:-new}.bin paper_2406_06022_b200/libgsb.so
timeout 900 python -m pytest tests/test_gpu_encoder.py tests/test_gpu_parity.py -x -q > gpurun_out/${T}_tests.log 2>&1; echo tests rc $?; tail -3 gpurun_out/${T}_tests.log
for v in ${VARS:-prev new prev new}; do
  cp scripts/libgsb_$v.bin paper_2406_06022_b200/libgsb.so
  timeout 600 python bench.py --config mag240m_1_16 --steps 200 --no-cpu-baseline > gpurun_out/${T}_b.log 2>&1
  python3 -c "
import json; l=json.loads(open('gpurun_out/${T}_b.log').read().strip().splitlines()[-1]); print('$v', round(l['ms_per_step'],4), l['phase_ms_alone'], {k:round(v['us_per_step'],1) for k,v in l['kernels'].items() if 'enc' in k})"
done
