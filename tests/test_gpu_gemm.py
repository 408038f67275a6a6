"""tcgen05 (3xTF32) GEMM modes against the oracle: the NC decoder exercises NN (logits),
NT (dh = dlogits Wc^T) and TN (dWc = h^T dlogits, dbc) with an odd class count (ragged N,
ragged K, padded rows); the RGCN layers exercise the grouped per-type slot stacks."""
import ctypes as C

import numpy as np
import pytest

import oracle
from tests._pair import close

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,d,Cn", [(300, 128, 349), (1024, 128, 8), (77, 64, 153), (129, 128, 256)])
def test_nc_loss_gemms(n, d, Cn):
    import torch
    from paper_2406_06022_b200 import build
    from paper_2406_06022_b200._lib import call
    build.build()
    rng = np.random.default_rng(n + Cn)
    h = rng.standard_normal((n, d)).astype(np.float32)
    Wc = (rng.standard_normal((d, Cn)) * 0.1).astype(np.float32)
    bc = rng.standard_normal(Cn).astype(np.float32)
    labels = rng.integers(0, Cn, n).astype(np.int32)
    seeds = np.arange(n, dtype=np.int64) + 5
    T = lambda a: torch.from_numpy(a).cuda()
    P = lambda x: C.c_void_p(x.data_ptr())
    hd, Wd, bd, ld, sd = T(h), T(Wc), T(bc), T(labels), T(seeds)
    ldl = (Cn + 3) // 4 * 4
    logits = torch.empty((n, ldl), device="cuda")
    rl = torch.zeros(n + 640, device="cuda")
    loss = torch.empty(1, device="cuda")
    dh = torch.empty((n, d), device="cuda")
    dW = torch.empty((d, Cn), device="cuda")
    db = torch.empty(Cn, device="cuda")
    call("gsb_nc_loss", P(hd), n, d, P(Wd), P(bd), Cn, P(ld), P(sd), 5, P(logits), P(rl), P(loss), P(dh), P(dW),
         P(db), None)
    torch.cuda.synchronize()
    l, lg, dh_r, dW_r, db_r = oracle.nc_loss(h, Wc, bc, labels)
    close(loss.cpu().numpy()[0], l, what="loss")
    close(dh.cpu().numpy(), dh_r, what="dh")
    close(dW.cpu().numpy(), dW_r, what="dWc")
    close(db.cpu().numpy(), db_r, what="dbc")
