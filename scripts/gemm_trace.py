"""Per-role timeline of CTA 0 of one TMA GEMM (GSB_GEMM_DBG=1024|knobs)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2406_06022_b200._lib import call  # noqa

P = lambda x: C.c_void_p(x.data_ptr())
M, K, N = int(os.environ.get("M", 1024)), 512, 128
A = torch.randn(M, K, device="cuda"); B = torch.randn(K, N, device="cuda"); out = torch.zeros(M, N, device="cuda")
for _ in range(3):
    call("gsb_gemm", 0, P(A), K, P(B), N, M, N, K, P(out), N, None)
torch.cuda.synchronize()
buf = np.zeros(256, np.uint64)
call("gsb_gemm_trace", buf.ctypes.data_as(C.c_void_p), 256)
tr = buf.reshape(4, 64).astype(np.int64)
t0 = tr[0, 63]
for r, name in enumerate(["producer", "mma", "split", "epi"]):
    v = [(x - t0) for x in tr[r, :17]]
    print(f"{os.environ.get('GSB_GEMM_DBG')} {name:9s}", " ".join(f"{x/1000:6.2f}" for x in v), "| start", (tr[r, 63] - t0) / 1000)
