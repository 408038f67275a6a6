# round 1 (third session) evidence: plain bench, launch list, one ncu --set full of the
# layer-0 aggregation and forward GEMM (eager step), all on one GPU
CMD="python bench.py --no-cpu-baseline --steps 10 --warmup 3 --profile-steps 2"
timeout 600 $CMD > gpurun_out/r1c_plain.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:'gsb::|cub::' -s 300 -c 300 --csv --log-file gpurun_out/r1c_launches.csv $CMD > gpurun_out/r1c_ncu_launch.log 2>&1; echo launches rc $?
CMD2="python bench.py --no-cpu-baseline --steps 3 --warmup 3 --profile-steps 1 --no-graph"
timeout 600 $CMD2 > gpurun_out/r1c_plain2.log 2>&1 && timeout 900 ncu --set full --import-source on --clock-control none -k regex:"agg_kernel|umma_gemm" -s 8 -c 4 -o gpurun_out/r1c_full $CMD2 > gpurun_out/r1c_ncu_full.log 2>&1; echo full rc $?
