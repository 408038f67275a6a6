. scripts/summ.sh
run() { n=$1; tag=$2; shift 2; timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus $n --no-cpu-baseline --steps 200 "$@" > gpurun_out/b48_$tag.log 2> gpurun_out/b48_$tag.err; echo "$tag rc $?"; summ gpurun_out/b48_$tag.log 2>/dev/null | head -4; }
run 1 mag1
run 2 mag2
run 4 mag4
run 1 1b1 --config synth_1b
run 2 1b2 --config synth_1b
run 4 1b4 --config synth_1b
