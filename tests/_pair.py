"""Builds the two independent sides of a parity test from the same seeded synthetic inputs:
the oracle (CPU, fp64, its own CSC) and the CUDA path (libgsb via the runtime driver).
Only `synth` is shared."""
from __future__ import annotations

import numpy as np

import oracle
import synth

RTOL_F32 = 1e-5   # BASELINE.json north_star: "relative tolerance of 1e-5 in fp32"


def close(gpu, ref, rtol=RTOL_F32, what=""):
    """|g - r| <= rtol*|r| + rtol*max|r|  (SURVEY §8(c) tolerance reading, DESIGN.md R-tol)."""
    g = np.asarray(gpu, dtype=np.float64)
    r = np.asarray(ref, dtype=np.float64)
    assert g.shape == r.shape, (what, g.shape, r.shape)
    if r.size == 0:
        return
    scale = np.abs(r).max()
    err = np.abs(g - r)
    bound = rtol * np.abs(r) + rtol * scale
    bad = err > bound
    assert not bad.any(), (f"{what}: {bad.sum()} / {r.size} outside tolerance; max err {err.max():.3e}, "
                           f"max|ref| {scale:.3e}, worst at {np.unravel_index(np.argmax(err - bound), r.shape)}")


def gpu_store(cfg, device="cuda", keep=None):
    import torch
    from paper_2406_06022_b200.runtime import GraphStore
    st = GraphStore(cfg.counts, cfg.etype_src(), cfg.etype_dst(), device)
    for r in range(cfg.num_etypes):
        s, d = synth.etype_coo(cfg, r, backend="torch", device=device)
        k = None if keep is None or r not in keep else torch.as_tensor(keep[r]).to(device)
        st.load_etype(r, s, d, k)
    for t in range(cfg.num_ntypes):
        st.set_features(t, synth.feature_table(cfg, t, backend="torch", device=device))
    return st


def oracle_graph(cfg, keep=None):
    return oracle.Graph(cfg, keep=keep)


def relu_tie_slack(res, R, layer, rtol=RTOL_F32):
    """Gradient slack from ambiguous ReLU decisions (DESIGN.md R-relutie).

    A pre-activation z whose oracle value lies within the forward tolerance of 0 may take
    either side of the ReLU on the GPU; flipping it changes dW[r][k][n] by at most
    |A_r[i][k] * dh[i][n]| and db[n] by |dh[i][n]| (first order, exact for one flip).
    Returns (slack_W (R+1, d_in, d_out), slack_b (d_out,), n_ambiguous)."""
    import oracle as _o
    z = res.zs[layer]
    dh = res.extra["dh"][layer]
    amb = np.abs(z) <= rtol * np.abs(z) + rtol * np.abs(z).max()
    blk = res.blocks[layer]
    h_src = res.extra["ins"][layer]
    A, c = _o.rgcn_means(blk, R, h_src)
    d_in = h_src.shape[1]
    d_out = z.shape[1]
    g = np.abs(dh) * amb
    sW = np.zeros((R + 1, d_in, d_out))
    for r in range(R):
        sW[r] = np.abs(A[:, r, :]).T @ g
    sW[R] = np.abs(h_src[blk.self_row]).T @ g
    return sW, g.sum(0), int(amb.sum())


def close_slack(gpu, ref, slack, rtol=RTOL_F32, what=""):
    g = np.asarray(gpu, dtype=np.float64)
    r = np.asarray(ref, dtype=np.float64)
    bound = rtol * np.abs(r) + rtol * np.abs(r).max() + slack
    bad = np.abs(g - r) > bound
    assert not bad.any(), f"{what}: {bad.sum()} / {r.size} outside tolerance (+ReLU-tie slack)"


def dsrc_tie_slack(res, R, layer, W, rtol=RTOL_F32):
    """Slack of a layer's input-row gradient dh_src from its ambiguous ReLU units (R-relutie):
    flipping unit (i, n) changes dZ[i, n] by dh[i, n], hence dh_src[u, k] by at most
    |dh[i, n] W_r[k, n]| / c_r(i) for every sampled edge u -> i of relation r, and by
    |dh[i, n] W_self[k, n]| for i's own source row (first order, exact for one flip)."""
    z = res.zs[layer]
    dh = res.extra["dh"][layer]
    amb = np.abs(z) <= rtol * np.abs(z) + rtol * np.abs(z).max()
    G = np.abs(dh) * amb
    blk = res.blocks[layer]
    Wa = np.abs(np.asarray(W, np.float64))
    out = np.zeros((len(blk.src_gid), Wa.shape[1]))
    for r in range(R):
        e = np.nonzero(blk.e_etype == r)[0]
        if len(e) == 0:
            continue
        M = G @ Wa[r].T
        np.add.at(out, blk.e_src[e], M[blk.e_dst[e]] / blk.seg_cnt[blk.e_dst[e], r][:, None])
    np.add.at(out, blk.self_row, G @ Wa[R].T)
    return out
