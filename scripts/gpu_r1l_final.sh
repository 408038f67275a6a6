# end of the fourth session: new multi-tile scan test, GPU suite, smoke, default bench, launch list
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k multi_tile > gpurun_out/r1l_multitile.log 2>&1; echo multitile rc $?; tail -2 gpurun_out/r1l_multitile.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r1l_tests.log 2>&1; echo tests rc $?; tail -2 gpurun_out/r1l_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1l_smoke.log 2>&1; echo smoke rc $?; tail -1 gpurun_out/r1l_smoke.log
timeout 600 python bench.py > gpurun_out/r1l_bench.log 2>&1; echo bench rc $?; tail -1 gpurun_out/r1l_bench.log | head -c 300; echo
