. scripts/summ.sh
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lp.py tests/test_gpu_gemm.py tests/test_gpu_multi.py -q -m gpu --tb=short -x 2>&1 | grep -E "Error|error|passed|failed|assert" | head -30
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/b31_mag1.log 2> gpurun_out/b31_mag1.err; echo mag1 rc $?; summ gpurun_out/b31_mag1.log; tail -3 gpurun_out/b31_mag1.err
timeout 300 python bench.py --no-cpu-baseline --feat-dtype bf16 > gpurun_out/b31_mag1bf.log 2> gpurun_out/b31_mag1bf.err; echo mag1-bf16 rc $?; summ gpurun_out/b31_mag1bf.log; tail -3 gpurun_out/b31_mag1bf.err
timeout 300 python bench.py --no-cpu-baseline --config synth_1b --steps 200 > gpurun_out/b31_1b.log 2> gpurun_out/b31_1b.err; echo 1b rc $?; summ gpurun_out/b31_1b.log; tail -3 gpurun_out/b31_1b.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29632 bench.py --gpus 2 --feat-dtype bf16 > gpurun_out/b31_mag2bf.log 2> gpurun_out/b31_mag2bf.err; echo mag2-bf16 rc $?; summ gpurun_out/b31_mag2bf.log; tail -3 gpurun_out/b31_mag2bf.err
