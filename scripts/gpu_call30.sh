. scripts/summ.sh
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lp.py -q -m gpu --tb=short -x 2>&1 | grep -E "Error|error|passed|failed|assert" | head -30
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/b30_mag1.log 2> gpurun_out/b30_mag1.err; echo mag1 rc $?; summ gpurun_out/b30_mag1.log; tail -3 gpurun_out/b30_mag1.err
timeout 300 python bench.py --no-cpu-baseline --pipeline off > gpurun_out/b30_mag1s.log 2> gpurun_out/b30_mag1s.err; echo mag1-serial rc $?; summ gpurun_out/b30_mag1s.log
timeout 300 python bench.py --no-cpu-baseline --config amazon_lp > gpurun_out/b30_lp.log 2> gpurun_out/b30_lp.err; echo lp rc $?; summ gpurun_out/b30_lp.log; tail -3 gpurun_out/b30_lp.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29632 bench.py --gpus 2 > gpurun_out/b30_mag2.log 2> gpurun_out/b30_mag2.err; echo mag2 rc $?; summ gpurun_out/b30_mag2.log; tail -3 gpurun_out/b30_mag2.err
