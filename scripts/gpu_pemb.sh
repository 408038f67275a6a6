# 2-GPU: MAG240M 1/16 with learnable author/institution tables partitioned over the ranks vs frozen
mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533"
timeout 600 $R bench.py --gpus 2 --config mag240m_1_16 --learnable-emb --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/pemb_learn.log 2>&1; echo learn rc $?
timeout 600 $R bench.py --gpus 2 --config mag240m_1_16 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/pemb_frozen.log 2>&1; echo frozen rc $?
for f in learn frozen; do tail -1 gpurun_out/pemb_$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['value'], d['ms_per_step'])"; done
