set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/chk_bench.log 2> gpurun_out/chk_bench.err; echo bench rc $?
tail -c 3000 gpurun_out/chk_bench.log; tail -5 gpurun_out/chk_bench.err
