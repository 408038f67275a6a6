CMD="python bench.py --steps 10 --warmup 3 --profile-steps 2 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain13.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:umma_gemm_kernel -s 20 -c 8 -o gpurun_out/prof_umma $CMD > gpurun_out/ncu13.log 2>&1; echo ncu rc $?
tail -3 gpurun_out/ncu13.log
