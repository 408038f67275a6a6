"""Micro-benchmark of the tcgen05 GEMMs (gsb_gemm: NN, NT, TN) at layer-like shapes.
Env: GSB_GEMM=umma|tma (kernel), GSB_GEMM_DBG (gemm_tma.cuh knobs)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_06022_b200 import build  # noqa
build.build()
from paper_2406_06022_b200._lib import call  # noqa

P = lambda x: C.c_void_p(x.data_ptr())
tag = f"gemm={os.environ.get('GSB_GEMM', 'tma')} dbg={os.environ.get('GSB_GEMM_DBG', '0')}"
SHAPES = [tuple(int(v) for v in x.split("x")) for x in os.environ.get("SHAPES", "16384x512x128,1024x512x128").split(",")]
for (M, K, N) in SHAPES:
    A = torch.randn(M, K, device="cuda")
    B = torch.randn(K, N, device="cuda")
    out = torch.zeros(M, N, device="cuda")
    A2 = torch.randn(M, N, device="cuda")
    o2 = torch.zeros(M, K, device="cuda")
    oW = torch.zeros(K, N, device="cuda")
    S = lambda: C.c_void_p(torch.cuda.current_stream().cuda_stream)
    fns = {0: lambda: call("gsb_gemm", 0, P(A), K, P(B), N, M, N, K, P(out), N, S()),        # C = A B
           1: lambda: call("gsb_gemm", 1, P(A2), N, P(B), N, M, N, K, P(o2), K, S()),        # C = A2 B^T
           2: lambda: call("gsb_gemm", 2, P(A), K, P(A2), N, M, N, K, P(oW), N, S())}        # C += A^T A2
    for mode, fn in fns.items():
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        # 20 launches captured in one CUDA graph: device time, no host enqueue cost
        g = torch.cuda.CUDAGraph()
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            with torch.cuda.graph(g, stream=st):
                for _ in range(20):
                    fn()
        torch.cuda.current_stream().wait_stream(st)
        g.replay()
        torch.cuda.synchronize()
        # correctness of one launch against fp64
        for x in (out, o2, oW):
            x.zero_()
        fn()
        torch.cuda.synchronize()
        ref = {0: A.double() @ B.double(), 1: A2.double() @ B.double().T, 2: A.double().T @ A2.double()}[mode]
        got = {0: out, 1: o2, 2: oW}[mode].double()
        rel = ((got - ref).norm() / ref.norm()).item()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 20 * 1e3
        fl = 2 * M * K * N
        print(f"{tag} mode={mode} M={M} K={K} N={N}: {us:8.1f} us  {fl / us / 1e6:7.1f} TFLOP/s  "
              f"A bytes {M * K * 4 / us / 1e3:7.1f} GB/s  rel err {rel:.2e}", flush=True)
