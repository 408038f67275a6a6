. scripts/summ.sh
timeout 900 python -m pytest tests/test_gpu_encoder.py -q -m gpu --tb=short 2>&1 | grep -E "Error|error|passed|failed|assert|outside" | head -30
timeout 600 ncu --set full --import-source on --clock-control none -k regex:enc_umma -c 2 -o gpurun_out/prof_enc python bench.py --no-cpu-baseline --config mag240m_1_16 --steps 2 --warmup 3 --profile-steps 1 --no-graph > gpurun_out/ncu_enc.log 2>&1; echo ncu rc $?; tail -3 gpurun_out/ncu_enc.log
