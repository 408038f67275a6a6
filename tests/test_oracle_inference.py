"""Oracle pins for full-graph layer-wise inference: a node's full-graph
embedding equals the mini-batch step's output for that node when every fanout is ALL (the
mini-batch computation is exact, not sampled), and the decoder's argmax.  CPU only."""
import numpy as np

import oracle
import synth


def test_full_graph_equals_all_fanout_minibatch():
    cfg = synth.scaled(synth.tiny(), 0.2, "tiny_fifth")
    cfg.fanouts = [-1, -1]
    og = oracle.Graph(cfg)
    params = {k: v.astype(np.float64) for k, v in synth.init_params(cfg).items()}
    hs = oracle.full_graph_infer(og, params)
    assert hs[-1].shape == (cfg.num_nodes, cfg.hidden)
    rng = np.random.default_rng(0)
    for t in range(cfg.num_ntypes):      # a few seeds per type (seeds grouped by type)
        seeds = np.sort(rng.choice(cfg.counts[t], 5, replace=False)) + cfg.node_off[t]
        res = oracle.nc_step(og, params, seeds, synth.labels(cfg), 0, cfg.rng_seed) \
            if t == cfg.target_ntype else None
        blocks = oracle.sample_blocks(og, seeds, cfg.fanouts, cfg.rng_seed, 0)
        h = oracle.gather(og, blocks[0].src_gid).astype(np.float64)
        for l in range(len(cfg.fanouts)):
            _, h = oracle.rgcn_fwd(blocks[l], og.R, h, params[f"W{l}"], params[f"b{l}"], relu=(l < 1))
        np.testing.assert_allclose(h, hs[-1][seeds], rtol=1e-12, atol=1e-12)
        if res is not None:
            np.testing.assert_allclose(res.hs[-1], hs[-1][seeds], rtol=1e-12, atol=1e-12)


def test_first_layer_is_mean_formula_on_a_node():
    """h_0[v] for one node written out from the CSC (R-rgcn, fanout ALL)."""
    cfg = synth.scaled(synth.tiny(), 0.1, "tiny_tenth")
    og = oracle.Graph(cfg)
    params = {k: v.astype(np.float64) for k, v in synth.init_params(cfg).items()}
    hs = oracle.full_graph_infer(og, params)
    F = {t: synth.feature_table(cfg, t).astype(np.float64) for t in range(cfg.num_ntypes)}
    W, b = params["W0"], params["b0"]
    slots = {t: [r for r in range(og.R) if og.dst_t[r] == t] for t in range(og.T)}
    for v_gid in (0, cfg.node_off[1] + 3, cfg.node_off[2] + 7):
        t = int(og.type_of(np.array([v_gid]))[0])
        v = v_gid - cfg.node_off[t]
        z = F[t][v] @ W[og.R] + b
        for r in slots[t]:
            nb = og.indices[r][og.indptr[r][v]:og.indptr[r][v + 1]]
            if len(nb):
                z += F[og.src_t[r]][nb].mean(0) @ W[r]
        np.testing.assert_allclose(hs[0][v_gid], np.maximum(z, 0), rtol=1e-12, atol=1e-12)


def test_nc_predict_argmax_and_ties():
    h = np.array([[1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])
    Wc = np.array([[2.0, 0.0, 1.0], [0.0, 2.0, 1.0]])
    bc = np.zeros(3)
    _, pred, margin = oracle.nc_predict(h, Wc, bc)
    assert list(pred) == [0, 1, 0]          # row 2: logits (2, 2, 2): lowest index on ties
    assert margin[2] == 0.0 and margin[0] == 1.0
