"""Time Eq. 1 feature construction (gsb_construct_features) on the MAG240M-shaped graph at
1/16 scale: every author's row = mean of its papers' 768-d bf16 rows (rev_writes in-edges).
Prints one JSON line: rows/s and algorithmic HBM GB/s (per in-edge one 1536-B source row + 4-B
index; per author 8-B indptr + 3072-B fp32 output row)."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import synth  # noqa: E402
from bench import build_gsb  # noqa: E402

cfg = synth.get("mag240m_1_16")
st, _ = build_gsb(cfg, torch.device("cuda"))
paper, author = cfg.ntypes.index("paper"), cfg.ntypes.index("author")
d = cfg.dim_of(paper)
n = int(cfg.counts[author])
rev = [r for r, e in enumerate(cfg.etypes) if e.src == paper and e.dst == author][0]
E = int(st.n_edges[rev])
chunk = 1 << 20
out = torch.empty((chunk, d), dtype=torch.float32, device="cuda")
from paper_2406_06022_b200._lib import call  # noqa: E402
import ctypes as C  # noqa: E402


def sweep():
    for a in range(0, n, chunk):
        c = min(chunk, n - a)
        call("gsb_construct_features", st.h, author, 1 << paper, a, c, C.c_void_p(out.data_ptr()), d, None)


sweep()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    sweep()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
alg = E * (d * 2 + 4) + n * (8 + d * 4)
print(json.dumps({"what": "Eq. 1 feature construction, authors from 768-d bf16 papers (mag240m 1/16)",
                  "authors": n, "in_edges": E, "ms": ms, "rows_per_s": n / ms * 1e3,
                  "alg_GBps": alg / ms / 1e6, "hbm_peak_GBps": 6554.2, "frac": alg / ms / 1e6 / 6554.2}))
