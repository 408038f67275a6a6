# full-size MAG240M-shaped N=4 A/B over prebuilt libgsb variants: bash scripts/gpu_bigab.sh TAG v1 v2 ...
T=$1; shift
for v in "$@"; do
  cp scripts/libgsb_$v.bin paper_2406_06022_b200/libgsb.so
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29515 \
     bench.py --gpus 4 --steps 100 --warmup 5 --config mag240m --no-cpu-baseline > gpurun_out/${T}_b.log 2>&1
  python3 -c "
import json; l=json.loads(open('gpurun_out/${T}_b.log').read().strip().splitlines()[-1]); print('$v', round(l['ms_per_step'],4), {k: round(v,4) for k,v in l['phase_ms_alone'].items()}, {k:round(v['us_per_step'],1) for k,v in l['kernels'].items() if 'enc' in k})"
done
