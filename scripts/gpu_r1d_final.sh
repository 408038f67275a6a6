# round 1 (fourth session) evidence for the current tree: GPU suite, smoke, default bench
# (with cpu_baseline), reference arm, synth_1b line, launch list, one ncu --set full capture
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1d_tests.log 2>&1; echo tests rc $?; tail -2 gpurun_out/r1d_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1d_smoke.log 2>&1; echo smoke rc $?
timeout 600 python bench.py > gpurun_out/r1d_bench.log 2>&1; echo bench rc $?; tail -1 gpurun_out/r1d_bench.log | head -c 600; echo
timeout 600 python bench.py --impl reference > gpurun_out/r1d_ref.log 2>&1; echo ref rc $?; tail -1 gpurun_out/r1d_ref.log | head -c 400; echo
timeout 300 python bench.py --no-cpu-baseline --config synth_1b --steps 300 > gpurun_out/r1d_1b.log 2>&1; echo 1b rc $?
CMD="python bench.py --no-cpu-baseline --steps 10 --warmup 3 --profile-steps 2"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:'gsb::|cub::' -s 300 -c 300 --csv --log-file gpurun_out/r1d_launches.csv $CMD > gpurun_out/r1d_ncu_launch.log 2>&1; echo launches rc $?
CMD2="python bench.py --no-cpu-baseline --steps 3 --warmup 3 --profile-steps 1 --no-graph"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"agg_kernel|umma_gemm" -s 8 -c 4 -o gpurun_out/r1d_full $CMD2 > gpurun_out/r1d_ncu_full.log 2>&1; echo full rc $?
