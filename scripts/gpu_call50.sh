. scripts/summ.sh
timeout 120 python -m pytest tests/test_gpu_gemm.py -q -m gpu --tb=short -x 2>&1 | grep -E "Error|error|passed|failed|assert|outside" | head -10
timeout 400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_lp.py tests/test_gpu_encoder.py -q -m gpu --tb=short -x 2>&1 | grep -E "Error|error|passed|failed|assert|outside" | head -30
timeout 200 python bench.py --no-cpu-baseline > gpurun_out/b50_mag1.log 2> gpurun_out/b50_mag1.err; echo mag1-512 rc $?; summ gpurun_out/b50_mag1.log; tail -3 gpurun_out/b50_mag1.err
GSB_SO=exp/libgsb_t256.so timeout 200 python bench.py --no-cpu-baseline > gpurun_out/b50_mag1b.log 2> gpurun_out/b50_mag1b.err; echo mag1-256 rc $?; summ gpurun_out/b50_mag1b.log
timeout 200 python bench.py --no-cpu-baseline --config amazon_lp > gpurun_out/b50_lp.log 2> gpurun_out/b50_lp.err; echo lp rc $?; summ gpurun_out/b50_lp.log
