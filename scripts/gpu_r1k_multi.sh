nvidia-smi --query-gpu=index,name --format=csv,noheader
timeout 900 python -m pytest tests/test_gpu_multi.py -q -m gpu --tb=short 2>&1 | tail -4
N=$(nvidia-smi --query-gpu=index --format=csv,noheader | wc -l)
for cfg in mag synth_1b; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --config $cfg --steps 200 --warmup 10 > gpurun_out/r1k_multi_${cfg}_$N.log 2> gpurun_out/r1k_multi_${cfg}_$N.err; echo rc $?
  python -c "import json; d=json.loads(open('gpurun_out/r1k_multi_${cfg}_$N.log').read().strip().splitlines()[-1]); print('$cfg N=$N', d['value'], d['ms_per_step'], d['e2e']['value'], d['config']['parallelism'])"
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus $N --config amazon_lp --neg local_joint --steps 50 --warmup 5 > gpurun_out/r1k_multi_lpl_$N.log 2> gpurun_out/r1k_multi_lpl_$N.err; echo rc $?
python -c "import json; d=json.loads(open('gpurun_out/r1k_multi_lpl_$N.log').read().strip().splitlines()[-1]); print('amazon local_joint N=$N', d['value'], d['ms_per_step'])"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus $N --config amazon_lp --neg joint --steps 50 --warmup 5 > gpurun_out/r1k_multi_lpj_$N.log 2> gpurun_out/r1k_multi_lpj_$N.err; echo rc $?
python -c "import json; d=json.loads(open('gpurun_out/r1k_multi_lpj_$N.log').read().strip().splitlines()[-1]); print('amazon joint N=$N', d['value'], d['ms_per_step'])"
