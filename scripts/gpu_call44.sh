. scripts/summ.sh
run() { tag=$1; shift; timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29700 + RANDOM % 200)) bench.py --gpus 4 --no-cpu-baseline --steps 200 "$@" > gpurun_out/b44_$tag.log 2> gpurun_out/b44_$tag.err; echo "$tag rc $?"; summ gpurun_out/b44_$tag.log | head -1; }
run f32u
run f32f --peer-gather fused
run bf16u --feat-dtype bf16
run bf16f --feat-dtype bf16 --peer-gather fused
run f32u_nopipe --pipeline off
