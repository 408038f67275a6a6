timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py tests/test_gpu_lp.py -q -m gpu 2>&1 | tail -15
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench9.log 2> gpurun_out/bench9.err; echo bench rc $?
tail -c 2500 gpurun_out/bench9.log; tail -3 gpurun_out/bench9.err
