for d in 0 1 2 3 4 6 7; do GSB_GEMM_DEBUG=$d timeout 120 python scripts/gemm_micro.py 2>&1 | grep dbg; done
