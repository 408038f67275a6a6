. scripts/summ.sh
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2406_06022_b200/csrc -I include scripts/probe_bf16.cu -o /tmp/probe_bf16 && timeout 60 /tmp/probe_bf16
timeout 900 python -m pytest tests/test_gpu_encoder.py -q -m gpu --tb=short -x 2>&1 | grep -E "Error|error|passed|failed|assert|outside" | head -30
timeout 600 python bench.py --no-cpu-baseline --config mag240m_1_16 --steps 100 > gpurun_out/b32_m240.log 2> gpurun_out/b32_m240.err; echo m240 rc $?; summ gpurun_out/b32_m240.log; tail -5 gpurun_out/b32_m240.err
