# multi-GPU evidence: partitioned-topology tests + bench lines.  usage: bash scripts/gpu_multi.sh TAG N [configs] [tests]
T=${1:-mg}; N=${2:-2}; CFGS=${3:-"mag synth_1b"}; TESTS=${4:-"tests/test_gpu_partitioned.py tests/test_gpu_multi.py"}
mkdir -p gpurun_out
python -c "from paper_2406_06022_b200 import build; build.build()" > gpurun_out/${T}_build.log 2>&1
if [ "$TESTS" != "none" ]; then
timeout 1200 python -m pytest $TESTS -q > gpurun_out/${T}_tests.log 2>&1; echo tests rc $?; tail -3 gpurun_out/${T}_tests.log
fi
. scripts/summ.sh
for c in $CFGS; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 \
     bench.py --gpus $N --steps 200 --warmup 10 --config $c > gpurun_out/${T}_bench_${c}_n$N.log 2>&1; echo bench $c rc $?
  summ gpurun_out/${T}_bench_${c}_n$N.log 2>/dev/null | head -4
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513 \
   bench.py --gpus $N --steps 50 --warmup 5 --config mag --sampling nccl > gpurun_out/${T}_bench_mag_nccl_n$N.log 2>&1; echo bench nccl rc $?
summ gpurun_out/${T}_bench_mag_nccl_n$N.log 2>/dev/null | head -4
