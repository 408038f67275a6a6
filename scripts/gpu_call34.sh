. scripts/summ.sh
timeout 900 python -m pytest tests/test_gpu_encoder.py -q -m gpu --tb=short 2>&1 | grep -E "Error|error|passed|failed|assert|outside" | head -30
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu --tb=short -x -k "nc_step or graph or pipelined" 2>&1 | grep -E "Error|error|passed|failed|assert|outside" | head -30
timeout 600 python bench.py --no-cpu-baseline --config mag240m_1_16 --steps 100 > gpurun_out/b34_m240.log 2> gpurun_out/b34_m240.err; echo m240 rc $?; summ gpurun_out/b34_m240.log; tail -3 gpurun_out/b34_m240.err
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/b34_mag1.log 2> gpurun_out/b34_mag1.err; echo mag1 rc $?; summ gpurun_out/b34_mag1.log; tail -3 gpurun_out/b34_mag1.err
