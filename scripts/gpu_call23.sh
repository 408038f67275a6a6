timeout 900 python -m pytest tests/test_gpu_lp.py -q -m gpu --tb=short 2>&1 | grep -E "Error|error|passed|failed" | head -20
timeout 900 python bench.py --config amazon_lp --steps 100 --no-cpu-baseline > gpurun_out/bench23_lp.log 2> gpurun_out/bench23_lp.err; echo lp rc $?
python -c "
import json
l=json.loads(open('gpurun_out/bench23_lp.log').read().strip().splitlines()[-1])
print('LP value',l['value'],l['unit'],'ms/step',l['ms_per_step'],'e2e',l['e2e']['value'])
for k,v in list(l['kernels'].items())[:12]: print(f'{k:22s} {v[\"us_per_step\"]:8.1f}')
"; tail -3 gpurun_out/bench23_lp.err
