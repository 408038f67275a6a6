set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu 2>&1 | tail -8
CMD="python bench.py --steps 20 --warmup 3 --profile-steps 2 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain3.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:"gsb::|cub::" -s 230 -c 200 --csv --log-file gpurun_out/launches3.csv $CMD > gpurun_out/ncu3.log 2>&1; echo ncu rc $?
timeout 600 $CMD > gpurun_out/plain3b.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:gemm_tn_kernel -s 6 -c 1 -o gpurun_out/prof_dW $CMD > gpurun_out/ncu3b.log 2>&1; echo ncu2 rc $?
ls -la gpurun_out
