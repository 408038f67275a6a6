"""Oracle pins for the negative samplers and score/loss variants of App. A:
uniform / local-joint / in-batch negatives, the dot-product score (Eq. 2) and the weighted
cross entropy (Eq. 5).  CPU only."""
import os
import zlib

import numpy as np
import pytest
import torch

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_uniform_negatives_count_range_and_keying():
    # K draws per training edge, N*K in total, all of dst_t
    N, K, n, base = 37, 5, 1000, 12345
    neg = oracle.uniform_negatives(N, K, n, base, seed=7, step=3)
    assert neg.shape == (N * K,)
    assert neg.min() >= base and neg.max() < base + n
    # draws are keyed by (global positive index, j, step): shifting pos_base re-labels rows
    tail = oracle.uniform_negatives(N - 10, K, n, base, seed=7, step=3, pos_base=10)
    np.testing.assert_array_equal(tail, neg[10 * K:])
    # a different step or seed gives different draws; uniform and joint streams are distinct
    assert (oracle.uniform_negatives(N, K, n, base, 7, 4) != neg).mean() > 0.9
    jn = oracle.joint_negatives(N, K, n, base, 7, 3)
    assert (jn[:K] != neg[:K]).any()


def test_uniform_negatives_chi2():
    # iid uniform over the dst type: chi-square over 16 buckets of the id range
    N, K, n = 4000, 8, 64
    neg = oracle.uniform_negatives(N, K, n, 0, seed=11, step=0)
    cnt = np.bincount(neg % 16, minlength=16)
    e = N * K / 16
    chi2 = ((cnt - e) ** 2 / e).sum()
    assert chi2 < 37.7       # p ~ 0.001 at 15 dof


def test_local_joint_stays_in_local_range():
    # local joint = joint sampling restricted to the local partition's nodes
    lo, cnt, base = 300, 250, 1000
    neg = oracle.joint_negatives(64, 8, cnt, base + lo, seed=5, step=1)
    assert neg.min() >= base + lo and neg.max() < base + lo + cnt
    # same groups share the same K nodes, as joint does
    g = neg.reshape(8, 8)
    full = oracle.joint_negatives(64, 8, cnt, 0, seed=5, step=1).reshape(8, 8)
    np.testing.assert_array_equal(g - (base + lo), full)


def _golden_inbatch():
    rows = {}
    for l in open(os.path.join(GOLDEN, "inbatch_example.txt")):
        if l.strip() and not l.startswith("#"):
            a, b = l.split(":")
            rows[int(a)] = [int(x) for x in b.split()]
    return rows


def test_in_batch_pairs_match_paper_example():
    # P:L358 worked example: with one-hot destinations the score of (u_i, v_j) reads off j
    ex = _golden_inbatch()
    B, d = 3, 3
    hu = np.ones((B, d))
    hv = np.eye(B) * np.array([1.0, 10.0, 100.0])[:, None]     # v_j scores 10^(j-1) against u = 1
    _, sc, *_ = oracle.lp_loss_ex(hu, hv, None, None, B - 1, 1, 1, 0)
    for i in range(B):
        assert sc[i, 0] == 10.0 ** i
        got = [int(round(np.log10(s))) + 1 for s in sc[i, 1:]]
        assert got == ex[i + 1]


def test_dot_product_score_closed_form():
    # Eq. 2: score = sum_k u_k x_k; small integers give exact values
    hu = np.array([[1.0, 2.0, 3.0], [0.0, -1.0, 2.0]])
    hv = np.array([[4.0, 5.0, 6.0], [1.0, 1.0, 1.0]])
    hn = np.array([[1.0, 0.0, 0.0], [0.0, 0.0, 2.0]])
    _, sc, *_ = oracle.lp_loss_ex(hu, hv, hn, None, 1, 1, 0, 0)   # uniform layout: row i = positive i
    np.testing.assert_array_equal(sc, [[32.0, 1.0], [1.0, 4.0]])
    # DistMult with rel = 1 equals the dot product (Eq. 3 -> Eq. 2)
    _, sc2, *_ = oracle.lp_loss_ex(hu, hv, hn, np.ones(3), 1, 1, 0, 0)
    np.testing.assert_array_equal(sc, sc2)


def test_weighted_ce_reduces_to_ce_and_drops_positive():
    rng = np.random.default_rng(3)
    B, K, d = 6, 3, 4
    hu, hv, hn, rel = rng.normal(size=(B, d)), rng.normal(size=(B, d)), rng.normal(size=(2 * K, d)), rng.normal(size=d)
    l1, *_ = oracle.lp_loss_ex(hu, hv, hn, rel, K, K, 0, 1)
    l2, *_ = oracle.lp_loss_ex(hu, hv, hn, rel, K, K, 0, 2, np.ones(B))
    assert abs(l1 - l2) < 1e-13
    # w = 0 removes the positive terms: the loss is the negatives' -ln(1 - sigma(s)) alone
    l0, sc, *_ = oracle.lp_loss_ex(hu, hv, hn, rel, K, K, 0, 2, np.zeros(B))
    ref = np.mean(np.log1p(np.exp(sc[:, 1:])).sum(1) / (K + 1))
    assert abs(l0 - ref) < 1e-12


@pytest.mark.parametrize("sampler,score,kind", [("uniform", "distmult", 0), ("uniform", "dot", 1),
                                                ("in_batch", "distmult", 0), ("in_batch", "dot", 1),
                                                ("joint", "dot", 2), ("in_batch", "distmult", 2)])
def test_lp_loss_ex_grads_vs_torch(sampler, score, kind):
    """Scores, loss and all gradients against torch autograd (library) for every layout."""
    rng = np.random.default_rng(zlib.crc32(f"{sampler}/{score}/{kind}".encode()))
    B, d = 8, 5
    K = B - 1 if sampler == "in_batch" else 3
    mode = 1 if sampler == "in_batch" else 0
    group = 1 if sampler == "uniform" else (K if sampler == "joint" else 1)
    n_hn = B * K if sampler == "uniform" else (-(-B // K) * K if sampler == "joint" else 0)
    hu, hv = rng.normal(size=(B, d)), rng.normal(size=(B, d))
    hn = rng.normal(size=(n_hn, d)) if mode == 0 else None
    rel = rng.normal(size=d) if score == "distmult" else None
    w = rng.uniform(0.2, 2.0, size=B) if kind == 2 else None
    loss, sc, dhu, dhv, dhn, drel = oracle.lp_loss_ex(hu, hv, hn, rel, K, group, mode, kind, w)
    U, V = torch.tensor(hu, requires_grad=True), torch.tensor(hv, requires_grad=True)
    N = torch.tensor(hn, requires_grad=True) if hn is not None else None
    R = torch.tensor(rel, requires_grad=True) if rel is not None else torch.ones(d, dtype=torch.float64)
    Ur = U * R
    pos = (Ur * V).sum(1)
    if mode == 0:
        idx = (torch.arange(B)[:, None] // group) * K + torch.arange(K)[None, :]
        neg = torch.einsum("bk,bjk->bj", Ur, N[idx])
    else:
        idx = torch.tensor([[j if j < i else j + 1 for j in range(K)] for i in range(B)])
        neg = torch.einsum("bk,bjk->bj", Ur, V[idx])
    S = torch.cat([pos[:, None], neg], 1)
    if kind == 0:
        L = (torch.logsumexp(S, 1) - pos).mean()
    else:
        y = torch.zeros_like(S); y[:, 0] = 1
        wt = torch.ones_like(S)
        if kind == 2:
            wt[:, 0] = torch.tensor(w)
        L = torch.nn.functional.binary_cross_entropy_with_logits(S, y, weight=wt, reduction="none").mean(1).mean()
    L.backward()
    np.testing.assert_allclose(sc, S.detach().numpy(), rtol=1e-12, atol=1e-13)
    assert abs(loss - L.item()) < 1e-12
    np.testing.assert_allclose(dhu, U.grad.numpy(), rtol=1e-11, atol=1e-13)
    np.testing.assert_allclose(dhv, V.grad.numpy(), rtol=1e-11, atol=1e-13)
    if N is not None:
        np.testing.assert_allclose(dhn, N.grad.numpy(), rtol=1e-11, atol=1e-13)
    if rel is not None:
        np.testing.assert_allclose(drel, R.grad.numpy(), rtol=1e-11, atol=1e-13)
