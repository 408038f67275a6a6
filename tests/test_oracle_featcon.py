"""Oracle pins for Eq. 1 feature construction of featureless nodes (SURVEY
§8(f) f4): F'_v = average of the featured in-neighbours' rows.  CPU only."""
import numpy as np

import oracle
import synth


def _graph(edges_by_rel, counts, src_t, dst_t):
    """Oracle graph from explicit COO lists (a hand-built heterograph)."""
    import dataclasses
    cfg = dataclasses.replace(synth.tiny(), ntypes=[f"t{t}" for t in range(len(counts))], counts=list(counts),
                              etypes=[synth.EType(f"r{r}", s, d, len(edges_by_rel[r]))
                                      for r, (s, d) in enumerate(zip(src_t, dst_t))])
    coo = {r: (np.array([a for a, _ in e], np.int64), np.array([b for _, b in e], np.int64))
           for r, e in enumerate(edges_by_rel)}
    return oracle.Graph(cfg, coo=coo)


def test_star_center_is_mean_of_leaves_and_isolated_is_zero():
    # ntype 0 = featured "paper" (4 nodes), ntype 1 = featureless "author" (3 nodes)
    # r0: paper -> author.  author 0 <- papers 0, 1, 3; author 1 <- paper 2 twice (multi-edge);
    # author 2 isolated
    g = _graph([[(0, 0), (1, 0), (3, 0), (2, 1), (2, 1)]], [4, 3], [0], [1])
    F = np.array([[1.0, 0.0], [2.0, 4.0], [8.0, -2.0], [3.0, 1.0]])
    out = oracle.construct_features(g, 1, [0], feats={0: F})
    np.testing.assert_allclose(out[0], [2.0, 5.0 / 3.0], rtol=1e-15)   # (1+2+3)/3, (0+4+1)/3
    np.testing.assert_array_equal(out[1], F[2])              # a multi-edge counts twice: mean is the row
    np.testing.assert_array_equal(out[2], [0.0, 0.0])        # no featured neighbour


def test_mean_over_all_relations_edges_counted_once_each():
    # two relations into ntype 1 from two featured types with the same width; and a relation
    # from a featureless type (ntype 1 -> 1) that must be ignored
    g = _graph([[(0, 0)], [(0, 0), (1, 0)], [(1, 0)]], [2, 2, 2], [0, 2, 1], [1, 1, 1])
    F0 = np.array([[3.0, 3.0], [0.0, 0.0]])
    F2 = np.array([[6.0, 0.0], [0.0, 9.0]])
    out = oracle.construct_features(g, 1, [0, 2], feats={0: F0, 2: F2})
    np.testing.assert_array_equal(out[0], [3.0, 4.0])        # (3+6+0)/3, (3+0+9)/3
    np.testing.assert_array_equal(out[1], [0.0, 0.0])


def test_constant_rows_and_linearity_on_tiny():
    cfg = synth.tiny()
    og = oracle.Graph(cfg)
    # ntype 1 (B) receives r1 from ntype 0 (A)
    n0 = cfg.counts[0]
    c = np.full((n0, cfg.feat_dim), 0.375)
    out = oracle.construct_features(og, 1, [0], feats={0: c}, count=200)
    has = np.diff(og.indptr[1])[:200] > 0
    np.testing.assert_array_equal(out[has], 0.375)           # mean of a constant is the constant
    rng = np.random.default_rng(0)
    X, Y = rng.normal(size=(n0, cfg.feat_dim)), rng.normal(size=(n0, cfg.feat_dim))
    a = oracle.construct_features(og, 1, [0], feats={0: 2 * X - Y}, count=200)
    b = 2 * oracle.construct_features(og, 1, [0], feats={0: X}, count=200) - \
        oracle.construct_features(og, 1, [0], feats={0: Y}, count=200)
    np.testing.assert_allclose(a, b, atol=1e-12)
