timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_encoder.py tests/test_gpu_sparse_emb.py tests/test_gpu_inference.py -x -q -m gpu 2>&1 | grep -E "Error|error|assert|FAILED|passed|failed" | head -5
for cfg in mag synth_1b; do
  timeout 600 python bench.py --no-cpu-baseline --config $cfg --steps 300 > gpurun_out/ce_${cfg}.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ce_${cfg}.log').read().strip().splitlines()[-1]); print('$cfg', d['value'], d['ms_per_step'], d['e2e']['value'], sorted(((round(v['us_per_step'],1),k) for k,v in d['kernels'].items()), reverse=True))"
done
