"""Pins for the oracle's integer parts: Philox, index mapping, CSC, Floyd, sampler, relabel.

Every check here is against something other than the oracle itself: published
known-answer vectors, exact arithmetic, exhaustive enumeration, hand traces from
SPEC.md / PAPER.md, and invariants of the definitions.
"""
import itertools
import math
import os
from collections import Counter

import numpy as np
import pytest

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- Philox (R-rng)
def test_philox_known_answer_vectors():
    rows = [l.split() for l in open(os.path.join(GOLDEN, "philox_kat.txt")) if l.strip() and not l.startswith("#")]
    assert len(rows) == 3
    for r in rows:
        ctr = [int(x, 16) for x in r[0:4]]
        key = [int(x, 16) for x in r[4:6]]
        exp = [int(x, 16) for x in r[6:10]]
        assert list(oracle.philox4x32_10(ctr, key)) == exp


def test_keyed_u64_word_order():
    # u64 = (out[1] << 32) | out[0] with key = (seed lo, seed hi)  (R-rng)
    o = oracle.philox4x32_10([1, 2, 3, 4], [0x89ABCDEF, 0x01234567])
    assert oracle.keyed_u64(0x0123456789ABCDEF, 1, 2, 3, 4) == (int(o[1]) << 32) | int(o[0])


# ---------------------------------------------------------------- index mapping
@pytest.mark.parametrize("n", [1, 2, 3, 5, 7, 10, 64, 1000, 1 << 31, (1 << 40) + 3])
def test_unif_index_boundaries(n):
    """idx(x) = floor(x n / 2^64): the smallest x mapping to k is ceil(k 2^64 / n)."""
    two64 = 1 << 64
    rng = np.random.default_rng(n % 1000)
    ks = {0, n - 1} | {int(k) for k in rng.integers(0, n, size=20)}
    for k in ks:
        x0 = -((-k * two64) // n)  # ceil
        assert oracle.unif_index(x0, n) == k
        if x0 > 0:
            assert oracle.unif_index(x0 - 1, n) == k - 1
    assert oracle.unif_index(two64 - 1, n) == n - 1
    assert oracle.unif_index(0, n) == 0


def test_unif_index_all_small_n_counts():
    """Exact preimage sizes: #{x : idx(x) = k} = ceil((k+1)2^64/n) - ceil(k 2^64/n), which
    differ by at most 1 across k: the mapping is uniform up to 1/2^64 (bias bound)."""
    two64 = 1 << 64
    for n in range(1, 65):
        sizes = [(-(-(k + 1) * two64 // n)) - (-(-k * two64 // n)) for k in range(n)]
        assert sum(sizes) == two64
        assert max(sizes) - min(sizes) <= 1
        # and the oracle agrees at every boundary
        for k in range(n):
            x0 = -(-k * two64 // n)
            assert oracle.unif_index(x0, n) == k


# ---------------------------------------------------------------- Floyd (exhaustive)
@pytest.mark.parametrize("n,f", [(4, 2), (5, 3), (6, 3), (7, 4), (8, 4), (6, 6), (5, 1)])
def test_floyd_exhaustive_uniform(n, f):
    """Enumerate every draw sequence t_i in [0, n-f+i]: each f-subset of [0,n) must appear
    exactly prod(n-f+i+1)/C(n,f) times -> uniform without replacement (R-wor)."""
    ranges = [range(n - f + i + 1) for i in range(f)]
    cnt = Counter()
    total = 0
    for draws in itertools.product(*ranges):
        s = oracle.floyd(n, f, list(draws))
        assert len(set(s.tolist())) == f and all(0 <= x < n for x in s)
        assert list(s) == sorted(s)
        cnt[tuple(s)] += 1
        total += 1
    assert len(cnt) == math.comb(n, f)
    assert set(cnt.values()) == {total // math.comb(n, f)}


# ---------------------------------------------------------------- CSC (R-csc)
def test_csc_invariants_and_multiset():
    rng = np.random.default_rng(0)
    n_src, n_dst, E = 50, 40, 3000
    s = rng.integers(0, n_src, E).astype(np.int32)
    d = rng.integers(0, n_dst, E).astype(np.int32)
    ip, ix = oracle.build_csc(n_dst, s, d)
    assert ip[0] == 0 and ip[-1] == E and np.all(np.diff(ip) >= 0)
    got = Counter()
    for v in range(n_dst):
        seg = ix[ip[v]:ip[v + 1]]
        assert np.all(np.diff(seg) >= 0), "segment sorted by src"
        for u in seg:
            got[(int(u), v)] += 1
    assert got == Counter(zip(s.tolist(), d.tolist()))


def test_csc_keep_mask_drops_edges():
    s = np.array([0, 1, 2, 0], np.int32)
    d = np.array([1, 1, 1, 0], np.int32)
    ip, ix = oracle.build_csc(2, s, d, keep=np.array([1, 0, 1, 1], np.uint8))
    assert ip.tolist() == [0, 1, 3] and ix.tolist() == [0, 0, 2]


# ---------------------------------------------------------------- sampler
def _mini_cfg(counts, etypes, fanouts=(5, 5)):
    return synth.Config(name="t", ntypes=[f"T{i}" for i in range(len(counts))], counts=list(counts),
                        etypes=[synth.EType(f"r{i}", a, b, 0) for i, (a, b) in enumerate(etypes)],
                        feat_dim=4, fanouts=list(fanouts), batch=1, hidden=4, num_classes=2, target_ntype=0)


def _graph(counts, etypes, coo):
    cfg = _mini_cfg(counts, etypes)
    for r, (s, d) in coo.items():
        cfg.etypes[r].num_edges = len(s)
    return oracle.Graph(cfg, coo={r: (np.asarray(s, np.int32), np.asarray(d, np.int32)) for r, (s, d) in coo.items()})


def test_sampler_degree_below_fanout_returns_all():
    # node with 3 in-edges, fanout 5 -> all 3
    g = _graph([4], [(0, 0)], {0: ([1, 2, 3], [0, 0, 0])})
    seg, es, ee, et, ed = oracle.sample_hop(g, np.array([0]), 5, seed=1, step=0, hop=1)
    assert seg[0, 0] == 3 and es.tolist() == [1, 2, 3] and ee.tolist() == [0, 1, 2]


def test_sampler_path_graph_hand_trace():
    # path a->b->c, seeds {c}, fanout [ALL, ALL]: layer-1 srcs {c, b}, layer-2 {c, b, a}
    a, b, c = 0, 1, 2
    g = _graph([3], [(0, 0)], {0: ([a, b], [b, c])})
    blocks = oracle.sample_blocks(g, np.array([c]), [-1, -1], seed=7, step=0)
    assert blocks[1].dst_gid.tolist() == [c] and blocks[1].src_gid.tolist() == [c, b]
    assert blocks[0].dst_gid.tolist() == [c, b] and blocks[0].src_gid.tolist() == [c, b, a]
    assert blocks[0].e_src.tolist() == [1, 2]  # b -> row 1 (into c), a -> row 2 (into b)
    assert blocks[0].self_row.tolist() == [0, 1]


def test_sampler_star_graph_counts():
    # star graph, fanout [1]: block has exactly |seeds| edges
    n_leaf = 20
    s = [0] * n_leaf          # hub 0 -> every leaf, plus leaf -> leaf edges for variety
    d = list(range(1, n_leaf + 1))
    s += list(range(2, n_leaf + 1)); d += list(range(1, n_leaf))
    g = _graph([n_leaf + 1], [(0, 0)], {0: (s, d)})
    seeds = np.arange(1, n_leaf + 1)
    seg, es, *_ = oracle.sample_hop(g, seeds, 1, seed=3, step=5, hop=1)
    assert len(es) == len(seeds) and seg.sum() == len(seeds)


def test_sampler_fanout_all_is_exact_neighborhood():
    rng = np.random.default_rng(1)
    s = rng.integers(0, 30, 400); d = rng.integers(0, 30, 400)
    g = _graph([30], [(0, 0)], {0: (s, d)})
    seeds = np.arange(30)
    seg, es, ee, et, ed = oracle.sample_hop(g, seeds, -1, seed=1, step=0, hop=1)
    got = Counter(zip(es.tolist(), ed.tolist()))
    assert got == Counter(zip(s.tolist(), d.tolist()))


def test_sampler_invariants_random_heterograph():
    """count = min(f, deg); every sampled edge exists; positions distinct and ascending;
    deterministic; different step -> different draws."""
    cfg = synth.scaled(synth.tiny(), 0.2)
    g = oracle.Graph(cfg)
    rng = np.random.default_rng(2)
    seeds = rng.choice(cfg.counts[0], 200, replace=False).astype(np.int64)
    for f in (1, 3, 5, 11):
        seg, es, ee, et, ed = oracle.sample_hop(g, seeds, f, seed=11, step=4, hop=2)
        off = 0
        for j, v in enumerate(seeds):
            for r in range(g.R):
                if g.dst_t[r] != 0:
                    assert seg[j, r] == 0
                    continue
                deg = g.indptr[r][v + 1] - g.indptr[r][v]
                assert seg[j, r] == min(f, deg)
                e = slice(off, off + seg[j, r])
                assert np.all(et[e] == r) and np.all(ed[e] == j)
                pos = ee[e] - g.indptr[r][v]
                assert np.all(np.diff(pos) > 0) and np.all((pos >= 0) & (pos < deg))
                assert np.all(g.indices[r][ee[e]] + g.node_off[g.src_t[r]] == es[e])
                off += seg[j, r]
        assert off == len(es)
        again = oracle.sample_hop(g, seeds, f, seed=11, step=4, hop=2)
        assert np.array_equal(again[1], es) and np.array_equal(again[2], ee)
    other = oracle.sample_hop(g, seeds, 3, seed=11, step=5, hop=2)
    base = oracle.sample_hop(g, seeds, 3, seed=11, step=4, hop=2)
    assert not np.array_equal(other[2], base[2])


def test_sampler_uniform_chi_square():
    """deg 6, f 3: over 60k destinations every 3-subset of positions has frequency 1/20
    (chi-square, p > 1e-3): pins Floyd + Philox + index mapping together (R-wor)."""
    n = 60000
    deg, f = 6, 3
    d = np.repeat(np.arange(n), deg)
    s = np.tile(np.arange(deg), n)
    g = _graph([n, deg], [(1, 0)], {0: (s, d)})
    seg, es, ee, et, ed = oracle.sample_hop(g, np.arange(n), f, seed=99, step=0, hop=1)
    pos = (ee - np.repeat(np.arange(n) * deg, f)).reshape(n, f)
    keys = Counter(map(tuple, pos.tolist()))
    assert len(keys) == math.comb(deg, f)
    exp = n / math.comb(deg, f)
    chi2 = sum((c - exp) ** 2 / exp for c in keys.values())
    from scipy.stats import chi2 as C2
    assert C2.sf(chi2, math.comb(deg, f) - 1) > 1e-3


def test_sampler_exclusion():
    """batch target edges (u,v) in r* and their reverses (v,u) in rev(r*) are never
    sampled, and deg' = deg - #excluded."""
    rng = np.random.default_rng(5)
    n = 40
    s = rng.integers(0, n, 600); d = rng.integers(0, n, 600)
    s = np.concatenate([s, [3, 3, 3]]); d = np.concatenate([d, [7, 7, 7]])  # parallel target edges
    g = _graph([n], [(0, 0), (0, 0)], {0: (s, d), 1: (d, s)})
    exu = np.array([3, 10]); exv = np.array([7, 11])
    seeds = np.arange(n)
    seg, es, ee, et, ed = oracle.sample_hop(g, seeds, -1, seed=1, step=0, hop=1, excl_u=exu, excl_v=exv,
                                            excl_etype=0, excl_rev=1)
    for (u, v) in zip(exu, exv):
        assert not np.any((et == 0) & (ed == v) & (es == u))
        assert not np.any((et == 1) & (ed == u) & (es == v))
    # deg' check for v = 7 in r0
    deg7 = int(np.sum(d == 7)); n37 = int(np.sum((d == 7) & (s == 3)))
    assert seg[7, 0] == deg7 - n37
    # with a fanout, still never sampled
    for f in (1, 2, 4):
        seg, es, ee, et, ed = oracle.sample_hop(g, seeds, f, seed=2, step=1, hop=1, excl_u=exu, excl_v=exv,
                                                excl_etype=0, excl_rev=1)
        for (u, v) in zip(exu, exv):
            assert not np.any((et == 0) & (ed == v) & (es == u))
            assert not np.any((et == 1) & (ed == u) & (es == v))


def test_relabel_invariants():
    """dst prefix per type, ascending-unique new srcs, every edge src resolves (R-relabel)."""
    cfg = synth.scaled(synth.tiny(), 0.2)
    g = oracle.Graph(cfg)
    rng = np.random.default_rng(3)
    seeds = rng.choice(cfg.counts[0], 100, replace=False).astype(np.int64)
    blocks = oracle.sample_blocks(g, seeds, [4, 6], seed=5, step=2)
    for blk in blocks:
        t_dst = g.type_of(blk.dst_gid)
        t_src = g.type_of(blk.src_gid)
        assert np.all(np.diff(t_src) >= 0), "src list grouped by ascending ntype"
        assert len(np.unique(blk.src_gid)) == len(blk.src_gid)
        for t in range(g.T):
            dst_t = blk.dst_gid[t_dst == t]
            src_t = blk.src_gid[t_src == t]
            assert np.array_equal(src_t[:len(dst_t)], dst_t)
            new = src_t[len(dst_t):]
            assert np.all(np.diff(new) > 0)
            exp_new = np.setdiff1d(blk.e_src_gid[g.type_of(blk.e_src_gid) == t], dst_t)
            assert np.array_equal(new, exp_new)
        assert np.array_equal(blk.src_gid[blk.e_src], blk.e_src_gid)
        assert np.array_equal(blk.src_gid[blk.self_row], blk.dst_gid)
    assert np.array_equal(blocks[0].dst_gid, blocks[1].src_gid)
    assert np.array_equal(blocks[1].dst_gid, seeds)


def test_gather_matches_generator_rows():
    cfg = synth.scaled(synth.tiny(), 0.1)
    g = oracle.Graph(cfg)
    gids = np.array([0, 5, cfg.node_off[1] + 3, cfg.node_off[2] + 1, cfg.node_off[3] - 1], np.int64)
    x = oracle.gather(g, gids)
    for i, gid in enumerate(gids):
        t = int(np.searchsorted(cfg.node_off, gid, side="right") - 1)
        assert np.array_equal(x[i], synth.feature_rows(cfg, t, [gid - cfg.node_off[t]])[0])


def test_joint_negatives_counts_sharing_uniformity():
    # N=4, K=2 -> 2 groups, 4 draws; groups differ; P:L356 N draws total
    neg = oracle.joint_negatives(4, 2, 1000, 0, seed=1, step=0)
    assert neg.shape == (4,)
    # partial last group draws a fresh K-set -> ceil(N/K)*K
    assert oracle.joint_negatives(5, 2, 1000, 0, 1, 0).shape == (6,)
    # gid_base offset, range
    neg = oracle.joint_negatives(4096, 32, 777, 1000, seed=3, step=9)
    assert neg.shape == (4096,) and neg.min() >= 1000 and neg.max() < 1777
    big = oracle.joint_negatives(200000, 40, 50, 0, seed=4, step=1)
    cnt = np.bincount(big, minlength=50)
    exp = len(big) / 50
    from scipy.stats import chi2 as C2
    assert C2.sf(((cnt - exp) ** 2 / exp).sum(), 49) > 1e-3
