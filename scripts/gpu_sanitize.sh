# compute-sanitizer memcheck / racecheck over small parity cases (tiny configs)
T=${1:-san}
python -c "from paper_2406_06022_b200 import build; build.build()" > gpurun_out/${T}_build.log 2>&1
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "tiny and not bf16" > gpurun_out/${T}_memcheck.log 2>&1; echo memcheck rc $?; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/${T}_memcheck.log | tail -3
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_gemm.py -x -q -k "1024" > gpurun_out/${T}_memcheck_gemm.log 2>&1; echo memcheck gemm rc $?; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/${T}_memcheck_gemm.log | tail -3
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -x -q -k "test_nc_step_parity and tiny-True" > gpurun_out/${T}_racecheck.log 2>&1; echo racecheck rc $?; grep -E "RACECHECK SUMMARY|ERROR SUMMARY|passed|failed" gpurun_out/${T}_racecheck.log | tail -3
