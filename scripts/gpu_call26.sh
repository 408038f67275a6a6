nvidia-smi --query-gpu=index,memory.used,memory.total --format=csv
timeout 900 python bench.py --config synth_1b --steps 100 --no-cpu-baseline > gpurun_out/b26_1b_n1.log 2> gpurun_out/b26_1b_n1.err; echo n1 rc $?
python -c "
import json
l=json.loads(open('gpurun_out/b26_1b_n1.log').read().strip().splitlines()[-1])
print('1B N=1 value',l['value'],'ms/step',l['ms_per_step'],'e2e',l['e2e']['value'],'setup',l['setup_s'], 'roof', l['roofline']['kernel'], l['roofline']['frac'])
for k,v in list(l['kernels'].items())[:10]: print(f'{k:22s} {v[\"us_per_step\"]:8.1f}')
"; tail -3 gpurun_out/b26_1b_n1.err
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus 2 --config synth_1b --steps 100 --warmup 5 > gpurun_out/b26_1b_n2.log 2> gpurun_out/b26_1b_n2.err; echo n2 rc $?
python -c "
import json
l=json.loads(open('gpurun_out/b26_1b_n2.log').read().strip().splitlines()[-1])
print('1B N=2 value',l['value'],'ms/step',l['ms_per_step'],'nvlink',l.get('nvlink_bytes_per_step_rank0'))
for k,v in list(l['kernels'].items())[:10]: print(f'{k:22s} {v[\"us_per_step\"]:8.1f}')
"; tail -3 gpurun_out/b26_1b_n2.err
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29614 bench.py --gpus 2 --config synth_1b --steps 100 --warmup 5 --replicate-features > gpurun_out/b26_1b_n2r.log 2> gpurun_out/b26_1b_n2r.err; echo n2r rc $?
python -c "
import json
l=json.loads(open('gpurun_out/b26_1b_n2r.log').read().strip().splitlines()[-1])
print('1B N=2 replicated value',l['value'],'ms/step',l['ms_per_step'])
"; tail -3 gpurun_out/b26_1b_n2r.err
