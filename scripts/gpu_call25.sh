timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py tests/test_gpu_lp.py -q -m gpu --tb=short 2>&1 | grep -E "Error|error|passed|failed" | head -20
timeout 600 python bench.py > gpurun_out/bench25.log 2> gpurun_out/bench25.err; echo bench rc $?
python -c "
import json
l=json.loads(open('gpurun_out/bench25.log').read().strip().splitlines()[-1])
print('value',l['value'],'ms/step',l['ms_per_step'],'e2e',l['e2e']['value'], 'roof', l['roofline'], 'cpu', l.get('cpu_baseline'))
for k,v in list(l['kernels'].items())[:25]: print(f'{k:22s} {v[\"us_per_step\"]:8.1f}')
"; tail -3 gpurun_out/bench25.err
