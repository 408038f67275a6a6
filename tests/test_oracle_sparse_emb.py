"""Oracle pins for learnable sparse embeddings of featureless nodes (P:L156
"GraphStorm by default adds learnable embeddings on author nodes"): H0 rows are table rows,
their gradients are dH0 rows (finite differences through the whole step), sparse Adagrad
equals torch.optim.Adagrad on the dense table with zero gradient elsewhere.  CPU only."""
import numpy as np
import torch

import oracle
import synth


def test_sparse_adagrad_step1_closed_form_and_vs_torch():
    rng = np.random.default_rng(2)
    N, d = 40, 6
    E0 = rng.normal(size=(N, d))
    rows = np.array([3, 17, 0, 39])
    g = rng.normal(size=(4, d))
    E, st = E0.copy(), np.zeros((N, d))
    lr, eps = 0.05, 1e-10
    oracle.sparse_adagrad(E, st, rows, g, lr, eps)
    # step 1: state = g^2, update = -lr * g / (|g| + eps)
    np.testing.assert_allclose(E[rows], E0[rows] - lr * g / (np.abs(g) + eps), rtol=1e-15)
    untouched = np.setdiff1d(np.arange(N), rows)
    np.testing.assert_array_equal(E[untouched], E0[untouched])
    # three steps vs torch.optim.Adagrad on the dense table (zero gradient rows do not move)
    T = torch.tensor(E0.copy(), requires_grad=True)
    opt = torch.optim.Adagrad([T], lr=lr, eps=eps)
    E, st = E0.copy(), np.zeros((N, d))
    for k in range(3):
        rk = rng.choice(N, 7, replace=False)
        gk = rng.normal(size=(7, d))
        oracle.sparse_adagrad(E, st, rk, gk, lr, eps)
        G = np.zeros((N, d))
        G[rk] = gk
        opt.zero_grad()
        T.grad = torch.tensor(G)
        opt.step()
    np.testing.assert_allclose(E, T.detach().numpy(), rtol=1e-13, atol=1e-15)


def test_embedding_gradient_is_dH0_rows_by_finite_differences():
    """d loss / d Emb_t[r] through the full NC step (encoder -> RGCN -> CE) equals the dH0 row
    of the input that reads row r; central differences in fp64."""
    cfg = synth.scaled(synth.tiny_enc(), 0.25, "tiny_enc_q")
    og = oracle.Graph(cfg)
    params = {k: v.astype(np.float64) for k, v in synth.init_params(cfg).items()}
    rng = np.random.default_rng(4)
    for t in (1, 2):
        params[f"Emb{t}"] = rng.normal(scale=0.3, size=(cfg.counts[t], cfg.feat_dim))
    seeds, labels = synth.nc_seeds(cfg, 0), synth.labels(cfg)
    res = oracle.nc_step(og, params, seeds, labels, 0, cfg.rng_seed)
    gr = oracle.emb_grads(og, params, res.blocks[0].src_gid, res.extra["dH0"])
    assert set(gr) == {1, 2} and len(gr[1][0]) > 0
    h = 1e-6
    for t in (1, 2):
        rows, g = gr[t]
        for (r, k) in [(0, 0), (len(rows) // 2, 5), (len(rows) - 1, cfg.feat_dim - 1)]:
            E = params[f"Emb{t}"]
            old = E[rows[r], k]
            E[rows[r], k] = old + h
            lp = oracle.nc_step(og, params, seeds, labels, 0, cfg.rng_seed).loss
            E[rows[r], k] = old - h
            lm = oracle.nc_step(og, params, seeds, labels, 0, cfg.rng_seed).loss
            E[rows[r], k] = old
            fd = (lp - lm) / (2 * h)
            assert abs(fd - g[r, k]) <= 1e-6 * max(1.0, abs(g[r, k])) + 1e-9, (t, r, k, fd, g[r, k])


def test_sparse_adagrad_dist_pins():
    """R-sparsedist: N ranks' sparse gradients -> one Adagrad step per touched row with the
    mean over ranks.  Pinned by (a) N = 1 equals sparse_adagrad, (b) N identical ranks equal
    one rank, (c) torch.optim.Adagrad on the dense table fed the mean of the ranks' dense
    gradients (zero rows elsewhere), over three steps with overlapping row sets."""
    rng = np.random.default_rng(11)
    N, d, lr, eps = 50, 8, 0.1, 1e-10
    E0 = rng.normal(size=(N, d))
    rows = np.array([4, 9, 33])
    g = rng.normal(size=(3, d))
    Ea, sa = E0.copy(), np.zeros((N, d))
    Eb, sb = E0.copy(), np.zeros((N, d))
    oracle.sparse_adagrad(Ea, sa, rows, g, lr, eps)
    oracle.sparse_adagrad_dist(Eb, sb, [rows], [g], lr, eps)
    assert np.array_equal(Ea, Eb) and np.array_equal(sa, sb)
    Ec, sc = E0.copy(), np.zeros((N, d))
    oracle.sparse_adagrad_dist(Ec, sc, [rows] * 4, [g] * 4, lr, eps)
    assert np.allclose(Ec, Ea, rtol=0, atol=1e-15) and np.allclose(sc, sa, rtol=0, atol=1e-15)

    W = 3
    E, st = E0.copy(), np.zeros((N, d))
    T = torch.tensor(E0.copy(), requires_grad=True)
    opt = torch.optim.Adagrad([T], lr=lr, eps=eps)
    for step in range(3):
        rr = [rng.choice(N, size=int(rng.integers(5, 20)), replace=False) for _ in range(W)]
        gg = [rng.normal(size=(len(r), d)) for r in rr]
        dense = np.zeros((N, d))
        for r, x in zip(rr, gg):
            dense[r] += x / W
        oracle.sparse_adagrad_dist(E, st, rr, gg, lr, eps)
        opt.zero_grad()
        T.grad = torch.tensor(dense)
        opt.step()
        assert np.allclose(E, T.detach().numpy(), rtol=1e-12, atol=1e-12), step
    untouched = np.setdiff1d(np.arange(N), np.concatenate(rr))
    assert untouched.size == 0 or np.isfinite(E[untouched]).all()
