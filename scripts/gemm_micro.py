"""Micro-benchmark of the tcgen05 GEMM utility (gsb_gemm) at layer-like shapes."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_06022_b200 import build  # noqa
build.build()
from paper_2406_06022_b200._lib import call  # noqa

P = lambda x: C.c_void_p(x.data_ptr())
for (M, K, N) in [(17920, 512, 128), (151552, 512, 128), (1024, 512, 128)]:
    A = torch.randn(M, K, device="cuda")
    B = torch.randn(K, N, device="cuda")
    out = torch.zeros(M, N, device="cuda")
    for mode in (0, 1):
        if mode == 1:
            Bm = torch.randn(K, N, device="cuda")   # C[M][K] = A[M][N] B[K][N]^T with N = 128 reduction
            A2 = torch.randn(M, N, device="cuda")
            o2 = torch.zeros(M, K, device="cuda")
            fn = lambda: call("gsb_gemm", 1, P(A2), N, P(Bm), N, M, N, K, P(o2), K, None)
        else:
            fn = lambda: call("gsb_gemm", 0, P(A), K, P(B), N, M, N, K, P(out), N, None)
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            fn()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 20 * 1e3
        fl = 2 * M * K * N
        print(f"dbg={os.environ.get('GSB_GEMM_DEBUG','0')} mode={mode} M={M} K={K} N={N}: {us:8.1f} us  "
              f"{fl / us / 1e6:7.1f} TFLOP/s  A bytes/us {M * K * 4 / us / 1e3:7.1f} GB/s", flush=True)
