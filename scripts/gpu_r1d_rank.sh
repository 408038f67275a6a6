# two-launch bitmap rank (rank_sum + rank_scan) replacing popc + CUB scan: GPU suite, bench mag/synth_1b, launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1e_tests.log 2>&1; echo tests rc $?; tail -2 gpurun_out/r1e_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1e_smoke.log 2>&1; echo smoke rc $?
for i in 1 2; do
timeout 600 python bench.py --no-cpu-baseline --steps 300 > gpurun_out/r1e_bench$i.log 2>&1; echo bench rc $?; tail -1 gpurun_out/r1e_bench$i.log | head -c 300; echo
timeout 300 python bench.py --no-cpu-baseline --config synth_1b --steps 300 > gpurun_out/r1e_1b$i.log 2>&1; echo 1b rc $?; tail -1 gpurun_out/r1e_1b$i.log | head -c 300; echo
done
CMD="python bench.py --no-cpu-baseline --steps 10 --warmup 3 --profile-steps 2"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base demangled -k regex:'gsb::|cub::' -s 300 -c 300 --csv --log-file gpurun_out/r1e_launches.csv $CMD > gpurun_out/r1e_ncu_launch.log 2>&1; echo launches rc $?
