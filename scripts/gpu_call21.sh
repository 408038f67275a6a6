CMD="python bench.py --steps 10 --warmup 3 --profile-steps 2 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain21.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:agg_kernel -s 4 -c 2 -o gpurun_out/prof_agg $CMD > gpurun_out/ncu21.log 2>&1; echo ncu rc $?
tail -2 gpurun_out/ncu21.log
