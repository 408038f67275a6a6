# big partitioned configs on N GPUs.  usage: bash scripts/gpu_big.sh TAG N CONFIG [steps]
T=$1; N=$2; C=$3; K=${4:-100}
python -c "from paper_2406_06022_b200 import build; build.build()" > /dev/null 2>&1
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29514 \
   bench.py --gpus $N --steps $K --warmup 5 --config $C --no-cpu-baseline > gpurun_out/${T}_bench_${C}_n$N.log 2>&1; echo bench $C rc $?
. scripts/summ.sh; summ gpurun_out/${T}_bench_${C}_n$N.log 2>/dev/null | head -4
python3 -c "
import json; l=json.loads(open('gpurun_out/${T}_bench_${C}_n$N.log').read().strip().splitlines()[-1]); print('setup_s', l['setup_s'], 'phases', l['phase_ms_alone'], 'nodes', l['config']['nodes'], 'edges', l['config']['edges'])" 2>/dev/null
tail -5 gpurun_out/${T}_bench_${C}_n$N.log | cut -c1-300
