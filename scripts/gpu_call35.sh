. scripts/summ.sh
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu --tb=short -x -k "nc_step" 2>&1 | grep -E "Error|error|passed|failed|assert|outside" | head -30
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/b35_mag1.log 2> gpurun_out/b35_mag1.err; echo mag1 rc $?; summ gpurun_out/b35_mag1.log; tail -3 gpurun_out/b35_mag1.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"enc_umma|nc_head|nc_dwc" -c 4 -o gpurun_out/prof_enc2 python bench.py --no-cpu-baseline --config mag240m_1_16 --steps 2 --warmup 3 --profile-steps 1 --no-graph > gpurun_out/ncu_enc2.log 2>&1; echo ncu rc $?; tail -2 gpurun_out/ncu_enc2.log
