"""Which elements of a ragged gsb_gemm are wrong (tools)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_06022_b200 import build  # noqa
build.build()
from paper_2406_06022_b200._lib import call  # noqa

P = lambda x: C.c_void_p(x.data_ptr())
T = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
for mode, M, K, N in [(0, 300, 64, 100), (0, 1000, 96, 349), (2, 300, 64, 100), (2, 4097, 160, 128), (0, 4097, 160, 128)]:
    rng = np.random.default_rng(1)
    if mode == 0:
        A, B = rng.standard_normal((M, K)).astype(np.float32), rng.standard_normal((K, N)).astype(np.float32)
        ref = A.astype(np.float64) @ B
        out = torch.zeros((M, N), device="cuda")
        a, b = T(A), T(B)
        call("gsb_gemm", 0, P(a), K, P(b), N, M, N, K, P(out), N, None)
    else:
        A, B = rng.standard_normal((M, K)).astype(np.float32), rng.standard_normal((M, N)).astype(np.float32)
        ref = A.astype(np.float64).T @ B
        out = torch.zeros((K, N), device="cuda")
        a, b = T(A), T(B)
        call("gsb_gemm", 2, P(a), K, P(b), N, M, N, K, P(out), N, None)
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    bad = np.abs(o - ref) > 1e-3 * (1 + np.abs(ref))
    rows = np.where(bad.any(1))[0]
    cols = np.where(bad.any(0))[0]
    print(os.environ.get("GSB_GEMM", "tma3"), mode, M, K, N, "bad", bad.sum(), "rows", rows[:5], rows[-3:] if len(rows) else None,
          "n rows", len(rows), "cols", cols[:5], cols[-3:] if len(cols) else None, "n cols", len(cols),
          "ratio sample", (o[bad][:3] / ref[bad][:3]) if bad.any() else None, flush=True)
