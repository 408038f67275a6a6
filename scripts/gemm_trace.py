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
for _ in range(300):
    call("gsb_gemm", 0, P(A), K, P(B), N, M, N, K, P(out), N, None)
torch.cuda.synchronize()
buf = np.zeros(256, np.uint64)
call("gsb_gemm_trace", buf.ctypes.data_as(C.c_void_p), 256)
tr = buf.reshape(4, 64).astype(np.int64)
t0 = tr[0, 63]
tag = f"M={M} dbg={os.environ.get('GSB_GEMM_DBG')}"
print(tag, "entry", (tr[0, 62] - t0) / 1000, "epi end after bulk wait", (tr[3, 62] - t0) / 1000)
if int(os.environ.get("GSB_GEMM_DBG", 0)) & 2048:
    print(tag, "producer top/after-wait/after-issue", " ".join(f"{(x - t0)/1000:.3f}" for x in tr[0, :36]))
for r, name in enumerate(["producer", "mma", "split"]):
    v = [(x - t0) for x in tr[r, :17]]
    print(tag, f"{name:9s}", " ".join(f"{x/1000:6.2f}" for x in v))
if int(os.environ.get("GSB_GEMM_DBG", 0)) & 4096:
    print(tag, "epi chunk0: ld/bias/waitread/sync1/sts/fence/sync2", " ".join(f"{(x - t0)/1000:.3f}" for x in tr[2, 32:39]))
print(tag, "epi (wake, chunk stores 0-3, tile done)", " ".join(f"{(tr[3, i] - t0)/1000:6.2f}" for i in range(6)))
