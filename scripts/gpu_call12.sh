timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_parity.py tests/test_gpu_lp.py -q -m gpu --tb=short 2>&1 | grep -E "Error|error|passed|failed" | head -20
CMD="python bench.py --steps 10 --warmup 3 --profile-steps 2 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain12.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:"gsb::|cub::" -s 120 -c 200 --csv --log-file gpurun_out/launches12.csv $CMD > gpurun_out/ncu12.log 2>&1; echo ncu rc $?
python scripts/launch_summary.py gpurun_out/launches12.csv
