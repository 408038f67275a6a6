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


@pytest.mark.parametrize("mode,M,K,N", [(0, 300, 64, 100), (0, 1000, 96, 349), (0, 4097, 160, 128),
                                        (1, 300, 64, 100), (1, 1000, 96, 349), (1, 4097, 160, 128),
                                        (2, 300, 64, 100), (2, 1000, 96, 349), (2, 4097, 160, 128)])
def test_gemm_modes_ragged(mode, M, K, N):
    """gsb_gemm (the layers' tcgen05 3xTF32 kernel, single group) on ragged shapes: row counts not
    a multiple of the 128-row tile, column counts not a multiple of 4 (row strides the TMA cannot
    address: per-thread epilogue stores / atomics, B through the cp.async kernel), against the
    product in fp64 (its definition) within R-tol."""
    import torch
    from paper_2406_06022_b200 import build
    from paper_2406_06022_b200._lib import call
    build.build()
    rng = np.random.default_rng(M + 7 * K + N + mode)
    P = lambda x: C.c_void_p(x.data_ptr())
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()
    if mode == 0:      # C[M][N] = A[M][K] B[K][N]
        A, B = rng.standard_normal((M, K)), rng.standard_normal((K, N))
        ref = A.astype(np.float32).astype(np.float64) @ B.astype(np.float32).astype(np.float64)
        out = torch.zeros((M, N), device="cuda")
        a, b = T(A), T(B)          # keep the device copies alive until the call has run
        call("gsb_gemm", 0, P(a), K, P(b), N, M, N, K, P(out), N, None)
    elif mode == 1:    # C[M][K] = A[M][N] B[K][N]^T
        A, B = rng.standard_normal((M, N)), rng.standard_normal((K, N))
        ref = A.astype(np.float32).astype(np.float64) @ B.astype(np.float32).astype(np.float64).T
        out = torch.zeros((M, K), device="cuda")
        a, b = T(A), T(B)
        call("gsb_gemm", 1, P(a), N, P(b), N, M, N, K, P(out), K, None)
    else:              # C[K][N] += A[M][K]^T B[M][N]
        A, B = rng.standard_normal((M, K)), rng.standard_normal((M, N))
        ref = A.astype(np.float32).astype(np.float64).T @ B.astype(np.float32).astype(np.float64)
        out = torch.zeros((K, N), device="cuda")
        a, b = T(A), T(B)
        call("gsb_gemm", 2, P(a), K, P(b), N, M, N, K, P(out), N, None)
    torch.cuda.synchronize()
    close(out.cpu().numpy(), ref, what=f"gemm mode {mode} {M}x{K}x{N}")


def _rna_tf32(x32):
    """Round-to-nearest (ties away) to tf32 by bit arithmetic on fp32 values."""
    b = x32.view(np.uint32).astype(np.uint64)
    return (((b + 0x1000) & 0xFFFFE000) & 0xFFFFFFFF).astype(np.uint32).view(np.float32)


def test_adam_split_images():
    """gsb_adam_step_split: the parameters are updated exactly as by gsb_adam_step, hi / lo are the
    round-to-nearest tf32 split of the new values (hi + lo = p to 2^-22), and the padded segment
    copies the split row by row with the padded stride."""
    import torch
    from paper_2406_06022_b200 import build
    from paper_2406_06022_b200._lib import call
    build.build()
    rng = np.random.default_rng(11)
    n, off, rows, cols, ld = 5003, 1000, 17, 99, 100
    p0 = rng.standard_normal(n).astype(np.float32)
    g = rng.standard_normal(n).astype(np.float32)
    m = (rng.standard_normal(n) * 0.1).astype(np.float32)
    v = np.abs(rng.standard_normal(n) * 0.1).astype(np.float32)
    T = lambda a: torch.from_numpy(a.copy()).cuda()
    P = lambda x: C.c_void_p(x.data_ptr())
    pa, ma, va = T(p0), T(m), T(v)
    pb, mb, vb = T(p0), T(m), T(v)
    gd = T(g)
    hi, lo = torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda")
    ph, pl = torch.zeros(rows * ld, device="cuda"), torch.zeros(rows * ld, device="cuda")
    call("gsb_adam_step", P(pa), P(gd), P(ma), P(va), n, 1e-2, 0.9, 0.999, 1e-8, 3, None, None)
    call("gsb_adam_step_split", P(pb), P(gd), P(mb), P(vb), n, 1e-2, 0.9, 0.999, 1e-8, 3, None, P(hi), P(lo),
         off, rows, cols, ld, P(ph), P(pl), None)
    torch.cuda.synchronize()
    pn = pb.cpu().numpy()
    assert np.array_equal(pa.cpu().numpy(), pn)
    h_ref = _rna_tf32(pn)
    l_ref = _rna_tf32((pn - h_ref).astype(np.float32))
    assert np.array_equal(hi.cpu().numpy(), h_ref) and np.array_equal(lo.cpu().numpy(), l_ref)
    assert np.all(np.abs(h_ref.astype(np.float64) + l_ref - pn) <= 2.0 ** -21 * np.abs(pn))
    seg = np.arange(rows * cols)
    r, c = seg // cols, seg % cols
    assert np.array_equal(ph.cpu().numpy()[r * ld + c], h_ref[off + seg])
    assert np.array_equal(pl.cpu().numpy()[r * ld + c], l_ref[off + seg])
