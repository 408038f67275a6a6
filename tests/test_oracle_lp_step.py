"""Pins for the oracle's link-prediction step composition (oracle.lp_step, §8(a) a3', a9, a10,
a11): the seed set (a9), the target-edge exclusion wired into sampling (a3'),
and the scatter of the score gradients dhu / dhv / dhn back into the seed rows before the
RGCN backward (Eq. 7).  These are checked against

  * a hand-worked 5-node heterograph with fanout ALL, where every sampled neighbourhood and
    every relabelled src list is written out by hand below;
  * torch autograd (library) of an independently written Eq. 3 + Eq. 7 loss over the top
    layer's seed rows, indexed through a gid -> row dict (not the oracle's searchsorted);
  * central finite differences of the whole step's loss in double w.r.t. entries of
    W0, W1, b0, b1 and rel.

CPU only."""
import numpy as np
import torch

import oracle
import synth
from synth import Config, EType

# ---------------------------------------------------------------------- hand-worked graph
# One ntype A with 5 nodes.  r0 "buys" A->A is the LP target etype (note the parallel edge
# 0->1); r1 "buys_rev" holds every r0 pair reversed (reverse etype, excluded too, R-excl).
R0 = [(0, 1), (1, 2), (2, 3), (3, 4), (0, 2), (4, 0), (0, 1)]
R1 = [(d, s) for s, d in R0]
POS = [(0, 1), (2, 3)]           # the batch's positive (u, v) edges of r0

# In-neighbours (src gids, ascending) of every dst per etype AFTER the exclusion of the batch
# positives: when sampling dst v in r0 every parallel u->v edge is hidden, and when sampling
# dst u in r1 every v->u edge is hidden (at every hop).  Worked by hand:
#   r0 in-edges: 0:[4]  1:[0,0] -> both hidden (pos (0,1))   2:[0,1]  3:[2] -> hidden (pos (2,3))  4:[3]
#   r1 in-edges: 0:[1,1,2] -> the 1->0 twins hidden (pos (0,1)); 1:[2]; 2:[3] -> hidden (pos (2,3));
#                3:[4]; 4:[0]
HAND_NBRS = {0: {0: [4], 1: [], 2: [0, 1], 3: [], 4: [3]},
             1: {0: [2], 1: [2], 2: [], 3: [4], 4: [0]}}


def _hand_cfg(K=2):
    return Config(name="hand5_lp", ntypes=["A"], counts=[5],
                  etypes=[EType("buys", 0, 0, len(R0)), EType("buys_rev", 0, 0, len(R1), reverse_of=0)],
                  feat_dim=8, fanouts=[-1, -1], batch=len(POS), hidden=4, num_classes=0, target_ntype=0,
                  task="lp", lp_etype=0, lp_rev_etype=1, num_neg=K)


def _hand_graph(cfg):
    coo = {0: (np.array([s for s, _ in R0]), np.array([d for _, d in R0])),
           1: (np.array([s for s, _ in R1]), np.array([d for _, d in R1]))}
    return oracle.Graph(cfg, coo=coo)


def _params(cfg):
    return {k: v.astype(np.float64) for k, v in synth.init_params(cfg).items()}


def test_hand_trace_seed_set_and_exclusion():
    """Seed set = ascending unique(u ∪ v ∪ negatives) (a9); every hop's sampled
    neighbourhoods (fanout ALL) equal the hand-worked table with the positives and their
    reverse twins hidden; src lists = dst prefix ++ ascending new sources (R-relabel)."""
    cfg = _hand_cfg()
    g = _hand_graph(cfg)
    u = np.array([p[0] for p in POS], np.int64)
    v = np.array([p[1] for p in POS], np.int64)
    for step in range(4):
        res = oracle.lp_step(g, _params(cfg), u, v, step, cfg.rng_seed)
        neg = res.extra["neg"]
        assert len(neg) == 2 and all(0 <= x < 5 for x in neg)      # one joint group of K = 2 draws
        assert res.extra["seeds"].tolist() == sorted(set(u.tolist()) | set(v.tolist()) | set(neg.tolist()))
        frontier = res.extra["seeds"].tolist()
        for blk in res.blocks[::-1]:                   # hop 1 (seeds) first
            assert blk.dst_gid.tolist() == frontier
            e = 0
            new = set()
            for j, d in enumerate(frontier):
                for r in (0, 1):
                    got = blk.e_src_gid[e:e + blk.seg_cnt[j, r]].tolist()
                    assert blk.e_etype[e:e + blk.seg_cnt[j, r]].tolist() == [r] * len(got)
                    assert sorted(got) == HAND_NBRS[r][d], (step, d, r, got)
                    e += blk.seg_cnt[j, r]
                    new |= set(got) - set(frontier)
            assert e == len(blk.e_src_gid)
            assert blk.src_gid.tolist() == frontier + sorted(new)
            frontier = blk.src_gid.tolist()


def _torch_top_loss(cfg, res, u, v, rel):
    """Eq. 3 DistMult + Eq. 7 contrastive loss (R-lpmean) with joint negatives (group g =
    i // K shares negatives g*K .. g*K+K-1), written from the paper over the top layer's seed
    rows; rows are found through a gid -> row dict of the top block's dst list."""
    top = res.blocks[-1]
    row = {int(x): i for i, x in enumerate(top.dst_gid)}
    H = torch.tensor(res.hs[-1], dtype=torch.float64, requires_grad=True)
    r = torch.tensor(rel, dtype=torch.float64)
    neg = res.extra["neg"]
    K = cfg.num_neg
    terms = []
    for i in range(len(u)):
        hu, hv = H[row[int(u[i])]], H[row[int(v[i])]]
        pos = (hu * r * hv).sum()
        g = i // K
        negs = torch.stack([(hu * r * H[row[int(neg[g * K + j])]]).sum() for j in range(K)])
        s = torch.cat([pos[None], negs])
        terms.append(-(pos - torch.logsumexp(s, 0)))
    L = torch.stack(terms).mean()
    L.backward()
    return float(L.detach()), H.grad.numpy()


def test_score_gradient_scatter_into_seed_rows():
    """The gradient reaching the top layer's seed rows (res.extra["dh"][L-1]) equals torch
    autograd of the independently written loss: a node that is a positive endpoint and a
    negative at once (or a negative twice) gets the sum of all its roles."""
    cfg = _hand_cfg(K=2)
    g = _hand_graph(cfg)
    u = np.array([p[0] for p in POS], np.int64)
    v = np.array([p[1] for p in POS], np.int64)
    p = _params(cfg)
    shared = 0
    for step in range(12):
        res = oracle.lp_step(g, p, u, v, step, cfg.rng_seed)
        neg = res.extra["neg"]
        shared += len(set(neg.tolist()) & (set(u.tolist()) | set(v.tolist()))) + (neg[0] == neg[1])
        L, dH = _torch_top_loss(cfg, res, u, v, p["rel"])
        assert abs(L - res.loss) <= 1e-12 * max(1.0, abs(L))
        np.testing.assert_allclose(res.extra["dh"][-1], dH, rtol=1e-10, atol=1e-13)
    assert shared > 0, "no step exercised a node with several roles"


def test_lp_step_sampled_graph_torch_scatter():
    """Same check on the sampled tiny LP graph (fanouts [5, 5], K = 16): many shared nodes."""
    cfg = synth.scaled(synth.tiny_lp(), 0.1)
    cfg.batch, cfg.num_neg = 64, 16
    g = oracle.Graph(cfg, keep={cfg.lp_etype: synth.lp_keep_mask(cfg), cfg.lp_rev_etype: synth.lp_keep_mask(cfg)})
    p = _params(cfg)
    u, v = synth.lp_train_edges(cfg, 0)
    res = oracle.lp_step(g, p, u, v, 0, cfg.rng_seed)
    L, dH = _torch_top_loss(cfg, res, u, v, p["rel"])
    assert abs(L - res.loss) <= 1e-12 * max(1.0, abs(L))
    np.testing.assert_allclose(res.extra["dh"][-1], dH, rtol=1e-10, atol=1e-13)


def test_lp_step_finite_differences():
    """Central differences in double (eps 1e-6) of the whole LP step's loss (negatives, seed
    set, exclusion-aware sampling, 2 RGCN layers, DistMult, Eq. 7) w.r.t. entries of W0, W1,
    b0, b1 and rel: the composed backward (scatter into seed rows, layer backward through
    the relabelled blocks) is the derivative of the composed forward."""
    cfg = synth.scaled(synth.tiny_lp(), 0.1)
    cfg.batch, cfg.num_neg = 32, 8
    g = oracle.Graph(cfg, keep={cfg.lp_etype: synth.lp_keep_mask(cfg), cfg.lp_rev_etype: synth.lp_keep_mask(cfg)})
    params = _params(cfg)
    u, v = synth.lp_train_edges(cfg, 1)
    res = oracle.lp_step(g, params, u, v, 1, cfg.rng_seed)
    rng = np.random.default_rng(7)
    eps = 1e-6
    for name in ("W0", "W1", "b0", "b1", "rel"):
        G = res.grads[name]
        big = np.argsort(-np.abs(G).ravel())[:3]
        idxs = [np.unravel_index(i, G.shape) for i in big] + \
               [tuple(int(rng.integers(0, s)) for s in G.shape) for _ in range(2)]
        for idx in idxs:
            pp = dict(params); pp[name] = params[name].copy(); pp[name][idx] += eps
            pm = dict(params); pm[name] = params[name].copy(); pm[name][idx] -= eps
            fd = (oracle.lp_step(g, pp, u, v, 1, cfg.rng_seed).loss -
                  oracle.lp_step(g, pm, u, v, 1, cfg.rng_seed).loss) / (2 * eps)
            assert abs(fd - G[idx]) <= 1e-6 * max(1.0, np.abs(G).max()) + 1e-4 * abs(G[idx]), (name, idx, fd, G[idx])
