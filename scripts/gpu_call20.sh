timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py tests/test_gpu_lp.py tests/test_gpu_multi.py -q -m gpu --tb=short 2>&1 | grep -E "Error|error|passed|failed" | head -20
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench20.log 2> gpurun_out/bench20.err; echo bench rc $?
python -c "
import json
l=json.loads(open('gpurun_out/bench20.log').read().strip().splitlines()[-1])
print('value',l['value'],'ms/step',l['ms_per_step'],'e2e',l['e2e']['value'], 'roof', l['roofline']['kernel'], l['roofline']['frac'])
for k,v in list(l['kernels'].items())[:12]: print(f'{k:22s} {v[\"us_per_step\"]:8.1f}')
"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 100 --warmup 5 > gpurun_out/bench20_n2.log 2> gpurun_out/bench20_n2.err; echo n2 rc $?
tail -5 gpurun_out/bench20_n2.err
python -c "
import json
l=json.loads(open('gpurun_out/bench20_n2.log').read().strip().splitlines()[-1])
print('N=2 value',l['value'],'ms/step',l['ms_per_step'],'nvlink',l.get('nvlink_bytes_per_step_rank0'))
for k,v in list(l['kernels'].items())[:8]: print(f'{k:22s} {v[\"us_per_step\"]:8.1f}')
"
