"""Probe the tcgen05 GEMM layouts with index-valued operands (debug aid)."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2406_06022_b200 import build  # noqa
build.build()
from paper_2406_06022_b200._lib import call  # noqa

P = lambda x: C.c_void_p(x.data_ptr())


def gemm(mode, A, B, M, N, K, C0=None):
    A = torch.from_numpy(np.ascontiguousarray(A, np.float32)).cuda()
    B = torch.from_numpy(np.ascontiguousarray(B, np.float32)).cuda()
    if mode == 0:
        out = torch.zeros((M, N), device="cuda"); ldc = N
    elif mode == 1:
        out = torch.zeros((M, K), device="cuda"); ldc = K
    else:
        out = torch.zeros((K, N), device="cuda"); ldc = N
    call("gsb_gemm", mode, P(A), A.shape[1], P(B), B.shape[1], M, N, K, P(out), ldc, None)
    torch.cuda.synchronize()
    return out.cpu().numpy()


np.set_printoptions(linewidth=200)
M = N = K = 128
I = np.eye(128, dtype=np.float32)
kk = np.tile(np.arange(128, dtype=np.float32)[:, None], (1, 128))   # kk[k][n] = k
nn = np.tile(np.arange(128, dtype=np.float32)[None, :], (128, 1))   # nn[k][n] = n
for name, mode in (("NN", 0), ("NT", 1), ("TN", 2)):
    print("=====", name)
    if mode == 0:
        # C = I @ B  -> should equal B
        c1 = gemm(0, I, kk, M, N, K); c2 = gemm(0, I, nn, M, N, K)
        print("C=I@kk (expect row index):\n", c1[:10, :10]); print("C=I@nn (expect col index):\n", c2[:10, :10])
        a1 = gemm(0, kk.T.copy(), I, M, N, K)   # A[m][k] = k ... C = A @ I = A -> C[m][n] = n
        print("C=A@I with A[m][k]=m:\n", gemm(0, nn.T.copy(), I, M, N, K)[:10, :10])
        print("C=A@I with A[m][k]=k:\n", a1[:10, :10])
        R = np.random.default_rng(0).standard_normal((128, 128)).astype(np.float32)
        R2 = np.random.default_rng(1).standard_normal((128, 128)).astype(np.float32)
        print("rand max err", np.abs(gemm(0, R, R2, M, N, K) - R.astype(np.float64) @ R2).max())
    elif mode == 1:
        # C[M][K] = A[M][N] B[K][N]^T ; A = I (M x N), B = kk (K x N): C[m][k] = B[k][m] = k
        print("C = I @ kk^T (expect col idx):\n", gemm(1, I, kk, M, N, K)[:10, :10])
        print("C = I @ nn^T (expect row idx):\n", gemm(1, I, nn, M, N, K)[:10, :10])
        R = np.random.default_rng(0).standard_normal((128, 128)).astype(np.float32)
        R2 = np.random.default_rng(1).standard_normal((128, 128)).astype(np.float32)
        print("rand max err", np.abs(gemm(1, R, R2, M, N, K) - R.astype(np.float64) @ R2.T).max())
    else:
        # C[K][N] = A[M][K]^T B[M][N]; A = I: C[k][n] = B[k][n]
        print("C = I^T @ kk (expect row idx):\n", gemm(2, I, kk, M, N, K)[:10, :10])
        print("C = I^T @ nn (expect col idx):\n", gemm(2, I, nn, M, N, K)[:10, :10])
        R = np.random.default_rng(0).standard_normal((128, 128)).astype(np.float32)
        R2 = np.random.default_rng(1).standard_normal((128, 128)).astype(np.float32)
        print("rand max err", np.abs(gemm(2, R, R2, M, N, K) - R.astype(np.float64).T @ R2).max())
