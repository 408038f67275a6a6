GSB_GEMM_DEBUG=1 timeout 120 python -m pytest tests/test_gpu_gemm.py -x -q -k "300" -s 2>&1 | grep gsb | head; 
GSB_GEMM_DEBUG=1 timeout 300 python bench.py --steps 5 --warmup 3 --profile-steps 1 --no-cpu-baseline 2>&1 | grep "\[gsb\]" | sort | uniq -c | head -20
