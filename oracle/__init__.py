"""CPU oracle for the RGCN mini-batch train step (GraphStorm, arXiv 2406.06022).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  It shares no code with
paper_2406_06022_b200/ (the CUDA product path); the only common module is `synth`
(seeded inputs, none of the method's arithmetic).

The arithmetic lives in oracle.c (plain C, fp64); this file marshals numpy arrays and
composes the steps of one train step in the paper's order (Fig. 4 P:L110-133,
Fig. 8): sample blocks hop by hop -> gather input features -> RGCN layers
(input layer first) -> loss -> backward (reverse order) -> optimizer.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (plain -O2; OpenMP only for oracle_set_threads > 1)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-fopenmp", "-shared", "-fPIC", "-o", _SO, _SRC,
                               "-lm"])
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_SO)
        P = C.c_void_p
        i64, i32, u64, u32, dbl = C.c_int64, C.c_int32, C.c_uint64, C.c_uint32, C.c_double
        sig = {
            "oracle_philox4x32_10": (None, [P, P, P]),
            "oracle_unif_index": (u64, [u64, u64]),
            "oracle_keyed_u64": (u64, [u64, u32, u32, u32, u32]),
            "oracle_build_csc": (i64, [i64, i64, P, P, P, P, P]),
            "oracle_floyd": (i64, [i64, i64, P]),
            "oracle_graph_new": (P, [i32, P, i32, P, P]),
            "oracle_graph_set_csc": (None, [P, i32, P, P]),
            "oracle_graph_free": (None, [P]),
            "oracle_sample_hop": (i64, [P, P, i64, i32, u64, u32, i32, P, P, i64, i32, i32, P, P, P, P, P, i64]),
            "oracle_relabel": (i64, [P, P, i64, P, i64, P, P, P, P, i64]),
            "oracle_gather": (None, [P, P, i32, P, i64, P]),
            "oracle_rgcn_means": (None, [i64, i32, i32, P, P, P, i64, P, P, P]),
            "oracle_rgcn_fwd": (None, [i64, i32, i32, i32, P, P, P, i64, P, P, P, P, i32, P, P]),
            "oracle_rgcn_bwd": (None, [i64, i64, i32, i32, i32, P, P, P, i64, P, P, P, P, i32, P, P, P, P]),
            "oracle_nc_loss": (dbl, [i64, i32, i32, P, P, P, P, P, P, P, P]),
            "oracle_joint_negatives": (i64, [i64, i32, i64, i64, u64, u32, i64, P]),
            "oracle_lp_loss": (dbl, [i64, i32, i32, P, P, P, P, i32, P, P, P, P, P]),
            "oracle_uniform_negatives": (i64, [i64, i32, i64, i64, u64, u32, i64, P]),
            "oracle_lp_loss_ex": (dbl, [i64, i32, i32, i32, i32, P, P, P, i64, P, i32, P, P, P, P, P, P]),
            "oracle_adam": (None, [i64, P, P, P, P, dbl, dbl, dbl, dbl, i32]),
            "oracle_sparse_adagrad": (None, [i64, i32, P, P, P, P, dbl, dbl]),
            "oracle_sgd": (None, [i64, P, P, dbl]),
            "oracle_set_threads": (None, [i32]),
            "oracle_max_threads": (i32, []),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def set_threads(n: int) -> None:
    """Threads of the layer loops (bit-identical results for any n; see oracle.c header)."""
    lib().oracle_set_threads(int(n))


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _c(a, dtype) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=dtype)


# ---------------------------------------------------------------------------------------
# primitives
# ---------------------------------------------------------------------------------------
def philox4x32_10(ctr, key) -> np.ndarray:
    c = _c(ctr, np.uint32)
    k = _c(key, np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    lib().oracle_philox4x32_10(_p(c), _p(k), _p(o))
    return o


def unif_index(x: int, n: int) -> int:
    return int(lib().oracle_unif_index(x, n))


def keyed_u64(seed: int, c0: int, c1: int, c2: int, c3: int) -> int:
    return int(lib().oracle_keyed_u64(seed, c0, c1, c2, c3))


def floyd(n: int, f: int, draws) -> np.ndarray:
    s = _c(draws, np.int64).copy()
    lib().oracle_floyd(n, f, _p(s))
    return s


def build_csc(n_dst: int, src: np.ndarray, dst: np.ndarray, keep: Optional[np.ndarray] = None):
    src = _c(src, np.int32)
    dst = _c(dst, np.int32)
    k = None if keep is None else _c(keep, np.uint8)
    indptr = np.zeros(n_dst + 1, dtype=np.int64)
    E = int(len(src) if keep is None else k.sum())
    indices = np.zeros(max(E, 1), dtype=np.int32)
    E2 = lib().oracle_build_csc(n_dst, len(src), _p(src), _p(dst), _p(k), _p(indptr), _p(indices))
    assert E2 == E
    return indptr, indices[:E]


class Graph:
    """Oracle graph store: per-etype CSC built by the oracle itself from the COO."""

    def __init__(self, cfg, coo: Optional[Dict[int, tuple]] = None, keep: Optional[Dict[int, np.ndarray]] = None):
        import synth
        self.cfg = cfg
        self.T = cfg.num_ntypes
        self.R = cfg.num_etypes
        self.node_off = cfg.node_off
        self.counts = np.asarray(cfg.counts, dtype=np.int64)
        self.src_t = cfg.etype_src()
        self.dst_t = cfg.etype_dst()
        self.h = lib().oracle_graph_new(self.T, _p(self.counts), self.R, _p(self.src_t), _p(self.dst_t))
        self.indptr: List[np.ndarray] = []
        self.indices: List[np.ndarray] = []
        for r in range(self.R):
            s, d = coo[r] if coo is not None and r in coo else synth.etype_coo(cfg, r)
            kp = keep.get(r) if keep else None
            ip, ix = build_csc(cfg.counts[self.dst_t[r]], s, d, kp)
            self.indptr.append(ip)
            self.indices.append(ix)
            lib().oracle_graph_set_csc(self.h, r, _p(ip), _p(ix))
        self.feats: List[Optional[np.ndarray]] = [None] * self.T

    def __del__(self):
        try:
            lib().oracle_graph_free(self.h)
        except Exception:
            pass

    def type_of(self, gid: np.ndarray) -> np.ndarray:
        return np.searchsorted(self.node_off, gid, side="right") - 1


@dataclass
class Block:
    """One message-flow block (P:L484 blocks[i]): dst = frontier, src = next frontier."""
    dst_gid: np.ndarray
    src_gid: np.ndarray
    seg_cnt: np.ndarray          # (n_dst, R)
    e_src_gid: np.ndarray
    e_eid: np.ndarray
    e_etype: np.ndarray
    e_dst: np.ndarray
    e_src: np.ndarray            # src row (int32)
    self_row: np.ndarray
    src_type_cnt: np.ndarray


def sample_hop(g: Graph, dst_gid: np.ndarray, fanout: int, seed: int, step: int, hop: int,
               excl_u=None, excl_v=None, excl_etype: int = -1, excl_rev: int = -1):
    dst_gid = _c(dst_gid, np.int64)
    n = len(dst_gid)
    cap = 0
    t = g.type_of(dst_gid)
    for r in range(g.R):
        m = t == g.dst_t[r]
        if m.any():
            loc = dst_gid[m] - g.node_off[g.dst_t[r]]
            deg = g.indptr[r][loc + 1] - g.indptr[r][loc]
            cap += int(deg.sum() if fanout < 0 else np.minimum(deg, fanout).sum())
    cap = max(cap, 1)
    seg = np.zeros(n * g.R, dtype=np.int64)
    es, ee, et, ed = (np.zeros(cap, np.int64), np.zeros(cap, np.int64), np.zeros(cap, np.int32), np.zeros(cap, np.int64))
    eu = _c(excl_u if excl_u is not None else np.zeros(0), np.int64)
    ev = _c(excl_v if excl_v is not None else np.zeros(0), np.int64)
    E = lib().oracle_sample_hop(g.h, _p(dst_gid), n, fanout, seed, step, hop, _p(eu), _p(ev), len(eu),
                                excl_etype, excl_rev, _p(seg), _p(es), _p(ee), _p(et), _p(ed), cap)
    assert E >= 0
    return seg.reshape(n, g.R), es[:E], ee[:E], et[:E], ed[:E]


def relabel(g: Graph, dst_gid: np.ndarray, e_src_gid: np.ndarray):
    dst_gid = _c(dst_gid, np.int64)
    e_src_gid = _c(e_src_gid, np.int64)
    n, E = len(dst_gid), len(e_src_gid)
    cap = n + E + 1
    src = np.zeros(cap, np.int64)
    erow = np.zeros(max(E, 1), np.int32)
    self_row = np.zeros(max(n, 1), np.int64)
    tc = np.zeros(g.T, np.int64)
    ns = lib().oracle_relabel(g.h, _p(dst_gid), n, _p(e_src_gid), E, _p(src), _p(erow), _p(self_row), _p(tc), cap)
    assert ns >= 0
    return src[:ns], erow[:E], self_row[:n], tc


def sample_blocks(g: Graph, seeds: np.ndarray, fanouts: List[int], seed: int, step: int,
                  excl_u=None, excl_v=None, excl_etype: int = -1, excl_rev: int = -1) -> List[Block]:
    """Blocks for L layers; returned input-layer first (blocks[0] is consumed first).
    Hop h (1-based from the seeds) uses fanout f[L-h] (R-fanout)."""
    L = len(fanouts)
    frontier = _c(seeds, np.int64)
    hops = []
    for h in range(1, L + 1):
        f = fanouts[L - h]
        seg, es, ee, et, ed = sample_hop(g, frontier, f, seed, step, h, excl_u, excl_v, excl_etype, excl_rev)
        src, erow, self_row, tc = relabel(g, frontier, es)
        hops.append(Block(frontier, src, seg, es, ee, et, ed, erow, self_row, tc))
        frontier = src
    return hops[::-1]


def gather(g: Graph, gids: np.ndarray) -> np.ndarray:
    import synth
    gids = _c(gids, np.int64)
    dim = g.cfg.feat_dim
    for t in range(g.T):
        if g.feats[t] is None:
            g.feats[t] = synth.feature_table(g.cfg, t)
    ptrs = (C.c_void_p * g.T)(*[f.ctypes.data for f in g.feats])
    out = np.zeros((len(gids), dim), np.float32)
    lib().oracle_gather(g.h, ptrs, dim, _p(gids), len(gids), _p(out))
    return out


def input_rows(g: Graph, t: int, local_ids: np.ndarray) -> np.ndarray:
    """Raw feature rows F_t[local_ids] (per-ntype width), widened to float64 (exact): from the
    materialised table if present, else from the generator's closed form row by row."""
    import synth
    ids = np.asarray(local_ids, np.int64)
    if g.feats[t] is not None:
        return g.feats[t][ids].astype(np.float64)
    return synth.feature_rows(g.cfg, t, ids).astype(np.float64)


def encoder_fwd(g: Graph, params: Dict[str, np.ndarray], gids: np.ndarray) -> np.ndarray:
    """Input encoder (§8(a) a6; "node input encoders handle node features"
    featureless nodes): H0[i] = F_t[local(i)] Win_t for an ntype t with a projection,
    H0[i] = F_t[local(i)] (frozen table of width feat_dim) otherwise.  fp64."""
    cfg = g.cfg
    gids = np.asarray(gids, np.int64)
    ty = g.type_of(gids)
    H0 = np.zeros((len(gids), cfg.feat_dim))
    for t in range(g.T):
        rows = np.nonzero(ty == t)[0]
        if len(rows) == 0:
            continue
        if f"Emb{t}" in params:   # learnable embedding table (§8(f) f1): H0 rows are its rows
            H0[rows] = np.asarray(params[f"Emb{t}"], np.float64)[gids[rows] - g.node_off[t]]
            continue
        X = input_rows(g, t, gids[rows] - g.node_off[t])
        H0[rows] = X @ params[f"Win{t}"].astype(np.float64) if cfg.project[t] else X
    return H0


def emb_grads(g: Graph, params: Dict[str, np.ndarray], gids: np.ndarray, dH0: np.ndarray):
    """Sparse gradients of the learnable embedding tables (§8(f) f1): H0[i] = Emb_t[local(i)]
    is a row copy, so dEmb_t[local(i)] = dH0[i] for every input row i of type t (input rows
    are unique, so no row is hit twice).  Returns {t: (local rows, gradient rows)}."""
    gids = np.asarray(gids, np.int64)
    ty = g.type_of(gids)
    out = {}
    for t in range(g.T):
        if f"Emb{t}" in params:
            rows = np.nonzero(ty == t)[0]
            out[t] = (gids[rows] - g.node_off[t], np.asarray(dH0, np.float64)[rows])
    return out


def sparse_adagrad(E: np.ndarray, state: np.ndarray, rows: np.ndarray, grad: np.ndarray, lr: float,
                   eps: float = 1e-10):
    """In place on float64 E, state: Adagrad on the touched rows only (R-sparseopt)."""
    rows = _c(rows, np.int64)
    grad = _c(grad, np.float64)
    assert E.dtype == np.float64 and state.dtype == np.float64 and E.flags.c_contiguous
    lib().oracle_sparse_adagrad(len(rows), E.shape[1], _p(rows), _p(grad), _p(E), _p(state), lr, eps)


def sparse_adagrad_dist(E: np.ndarray, state: np.ndarray, rows_per_rank, grads_per_rank, lr: float,
                        eps: float = 1e-10):
    """Data-parallel sparse update of a table partitioned over N ranks (§8(f) f1 with §8(e);
    reading R-sparsedist): the gradient of row x is the mean over ranks of the rank's dEmb row
    (a rank that did not touch x contributes 0; dense gradients are mean-all-reduced the same
    way), and each touched row takes ONE Adagrad step (sparse_adagrad) with it.  Row
    ownership does not enter the result.  rows_per_rank[r]: distinct local rows of rank r."""
    N = len(rows_per_rank)
    acc: Dict[int, np.ndarray] = {}
    for rows, grads in zip(rows_per_rank, grads_per_rank):
        rows = np.asarray(rows, np.int64)
        assert len(np.unique(rows)) == len(rows)
        for x, gr in zip(rows, np.asarray(grads, np.float64)):
            acc[int(x)] = acc.get(int(x), 0.0) + gr
    if not acc:
        return
    touched = np.array(sorted(acc), np.int64)
    g = np.stack([acc[int(x)] / N for x in touched])
    sparse_adagrad(E, state, touched, g, lr, eps)


def encoder_bwd(g: Graph, params: Dict[str, np.ndarray], gids: np.ndarray, dH0: np.ndarray) -> Dict[str, np.ndarray]:
    """dWin_t = sum over input rows i of type t of F_t[local(i)]^T dH0[i] (H0 = X Win_t is
    linear in Win_t); frozen tables get no gradient."""
    cfg = g.cfg
    gids = np.asarray(gids, np.int64)
    ty = g.type_of(gids)
    out = {}
    for t in range(g.T):
        if not cfg.project[t]:
            continue
        rows = np.nonzero(ty == t)[0]
        X = input_rows(g, t, gids[rows] - g.node_off[t])
        out[f"Win{t}"] = X.T @ np.asarray(dH0, np.float64)[rows]
    return out


def rgcn_fwd(blk: Block, R: int, h_src: np.ndarray, W: np.ndarray, b: np.ndarray, relu: bool):
    h_src = _c(h_src, np.float64)
    W = _c(W, np.float64)
    b = _c(b, np.float64)
    n = len(blk.dst_gid)
    d_in, d_out = W.shape[1], W.shape[2]
    z = np.zeros((n, d_out))
    h = np.zeros((n, d_out))
    lib().oracle_rgcn_fwd(n, R, d_in, d_out, _p(_c(blk.e_dst, np.int64)), _p(_c(blk.e_etype, np.int32)),
                          _p(_c(blk.e_src, np.int32)), len(blk.e_dst), _p(_c(blk.self_row, np.int64)),
                          _p(h_src), _p(W), _p(b), int(relu), _p(z), _p(h))
    return z, h


def rgcn_means(blk: Block, R: int, h_src):
    """Per-relation sampled means A (n_dst, R, d_in) and counts c (n_dst, R)."""
    h_src = _c(h_src, np.float64)
    n = len(blk.dst_gid)
    d_in = h_src.shape[1]
    c = np.zeros((n, R), np.int64)
    A = np.zeros((n, R, d_in))
    lib().oracle_rgcn_means(n, R, d_in, _p(_c(blk.e_dst, np.int64)), _p(_c(blk.e_etype, np.int32)),
                            _p(_c(blk.e_src, np.int32)), len(blk.e_dst), _p(h_src), _p(c), _p(A))
    return A, c


def rgcn_bwd(blk: Block, R: int, h_src, W, z, relu: bool, dh_dst, need_dh_src: bool):
    h_src = _c(h_src, np.float64)
    W = _c(W, np.float64)
    z = _c(z, np.float64)
    dh_dst = _c(dh_dst, np.float64)
    n = len(blk.dst_gid)
    n_src = len(blk.src_gid)
    d_in, d_out = W.shape[1], W.shape[2]
    dW = np.zeros_like(W)
    db = np.zeros(d_out)
    dhs = np.zeros((n_src, d_in)) if need_dh_src else None
    lib().oracle_rgcn_bwd(n, n_src, R, d_in, d_out, _p(_c(blk.e_dst, np.int64)), _p(_c(blk.e_etype, np.int32)),
                          _p(_c(blk.e_src, np.int32)), len(blk.e_dst), _p(_c(blk.self_row, np.int64)),
                          _p(h_src), _p(W), _p(z), int(relu), _p(dh_dst), _p(dW), _p(db), _p(dhs))
    return dW, db, dhs


def nc_loss(h, Wc, bc, y, need_grads: bool = True):
    h = _c(h, np.float64)
    Wc = _c(Wc, np.float64)
    bc = _c(bc, np.float64)
    y = _c(y, np.int32)
    n, d = h.shape
    Cn = Wc.shape[1]
    logits = np.zeros((n, Cn))
    dh = np.zeros_like(h) if need_grads else None
    dWc = np.zeros_like(Wc) if need_grads else None
    dbc = np.zeros_like(bc) if need_grads else None
    loss = lib().oracle_nc_loss(n, d, Cn, _p(h), _p(Wc), _p(bc), _p(y), _p(logits), _p(dh), _p(dWc), _p(dbc))
    return loss, logits, dh, dWc, dbc


def construct_features(g: Graph, ntype: int, featured, feats=None, first: int = 0, count: Optional[int] = None):
    """Eq. 1 with f = average (R-eq1): for node v of the featureless ntype,
    F'_v = mean of F_u over every in-edge u -> v (every stored etype r with dst_t = ntype
    whose src type is in `featured`), each edge counted once; 0 when v has no such edge.
    feats[t]: float array (N_t, dim) of ntype t's rows (default: the generator's table).
    Returns float64 (count, dim) for local ids [first, first + count).  Plain loops."""
    import synth
    count = g.counts[ntype] - first if count is None else count
    feats = {t: (feats[t] if feats is not None and t in feats else synth.feature_table(g.cfg, t)) for t in featured}
    dim = feats[featured[0]].shape[1]
    rels = [r for r in range(g.R) if g.dst_t[r] == ntype and g.src_t[r] in featured]
    out = np.zeros((count, dim))
    for i in range(count):
        v = first + i
        acc, n = np.zeros(dim), 0
        for r in rels:
            for e in range(g.indptr[r][v], g.indptr[r][v + 1]):
                acc += feats[g.src_t[r]][g.indices[r][e]].astype(np.float64)
                n += 1
        if n:
            out[i] = acc / n
    return out


def joint_negatives(n_pos: int, K: int, n_dst_nodes: int, gid_base: int, seed: int, step: int, group_base: int = 0):
    G = (n_pos + K - 1) // K
    neg = np.zeros(G * K, np.int64)
    lib().oracle_joint_negatives(n_pos, K, n_dst_nodes, gid_base, seed, step, group_base, _p(neg))
    return neg


def lp_loss(hu, hv, hn, rel, K: int, loss_kind: int = 0):
    hu, hv, hn, rel = (_c(x, np.float64) for x in (hu, hv, hn, rel))
    B, d = hu.shape
    G = (B + K - 1) // K
    scores = np.zeros((B, K + 1))
    dhu, dhv, dhn, drel = np.zeros_like(hu), np.zeros_like(hv), np.zeros((G * K, d)), np.zeros(d)
    loss = lib().oracle_lp_loss(B, K, d, _p(hu), _p(hv), _p(hn), _p(rel), loss_kind, _p(scores),
                                _p(dhu), _p(dhv), _p(dhn), _p(drel))
    return loss, scores, dhu, dhv, dhn, drel


def uniform_negatives(n_pos: int, K: int, n_dst_nodes: int, gid_base: int, seed: int, step: int,
                      pos_base: int = 0):
    """Uniform negatives (App. A.2.1): K iid draws per positive, n_pos*K in total."""
    neg = np.zeros(n_pos * K, np.int64)
    lib().oracle_uniform_negatives(n_pos, K, n_dst_nodes, gid_base, seed, step, pos_base, _p(neg))
    return neg


# negative samplers (App. A.2.1): name -> (mode, group(K)) for oracle_lp_loss_ex
NEG_SAMPLERS = ("joint", "uniform", "local_joint", "in_batch")


def lp_loss_ex(hu, hv, hn, rel, K: int, group: int, mode: int, loss_kind: int = 0, w=None):
    """General LP score + loss (oracle_lp_loss_ex): mode 0 = sampled negatives shared by
    `group` positives (hn rows), mode 1 = in-batch (K = B-1, hn unused); rel None = dot
    product (Eq. 2); loss_kind 2 = weighted CE with per-positive weights w."""
    hu, hv = _c(hu, np.float64), _c(hv, np.float64)
    B, d = hu.shape
    hn = _c(hn, np.float64) if mode == 0 else None
    n_hn = hn.shape[0] if hn is not None else 0
    rel = _c(rel, np.float64) if rel is not None else None
    w = _c(w, np.float64) if w is not None else None
    scores = np.zeros((B, K + 1))
    dhu, dhv = np.zeros_like(hu), np.zeros_like(hv)
    dhn = np.zeros((n_hn, d)) if hn is not None else None
    drel = np.zeros(d) if rel is not None else None
    loss = lib().oracle_lp_loss_ex(B, K, group, mode, d, _p(hu), _p(hv), _p(hn), n_hn, _p(rel), loss_kind, _p(w),
                                   _p(scores), _p(dhu), _p(dhv), _p(dhn), _p(drel))
    return loss, scores, dhu, dhv, dhn, drel


def adam(p, g, m, v, lr, t, b1=0.9, b2=0.999, eps=1e-8):
    """In place on float64 arrays p, m, v."""
    g = _c(g, np.float64)
    assert p.dtype == np.float64 and m.dtype == np.float64 and v.dtype == np.float64
    lib().oracle_adam(p.size, _p(p), _p(g), _p(m), _p(v), lr, b1, b2, eps, t)


# ---------------------------------------------------------------------------------------
# composition: one NC / LP train step in the paper's order
# ---------------------------------------------------------------------------------------
@dataclass
class StepResult:
    loss: float
    blocks: List[Block]
    x0: np.ndarray
    hs: List[np.ndarray]                 # layer outputs (h'), input-layer first
    zs: List[np.ndarray]
    grads: Dict[str, np.ndarray]
    extra: Dict[str, np.ndarray] = field(default_factory=dict)


def nc_step(g: Graph, params: Dict[str, np.ndarray], seeds: np.ndarray, labels: np.ndarray,
            step: int, rng_seed: int) -> StepResult:
    """Forward + backward of one NC mini-batch (no optimizer)."""
    cfg = g.cfg
    L = len(cfg.fanouts)
    blocks = sample_blocks(g, seeds, cfg.fanouts, rng_seed, step)
    if cfg.has_encoder:      # a6: projected / frozen input rows
        x0 = None
        h = encoder_fwd(g, params, blocks[0].src_gid)
    else:
        x0 = gather(g, blocks[0].src_gid)
        h = x0.astype(np.float64)
    hs, zs, ins = [], [], []
    for l in range(L):
        ins.append(h)
        z, h = rgcn_fwd(blocks[l], g.R, h, params[f"W{l}"], params[f"b{l}"], relu=(l < L - 1))
        zs.append(z)
        hs.append(h)
    y = labels[seeds - g.node_off[cfg.target_ntype]]
    loss, logits, dh, dWc, dbc = nc_loss(h, params["Wc"], params["bc"], y)
    grads = {"Wc": dWc, "bc": dbc}
    dhs = [None] * L
    for l in reversed(range(L)):
        dhs[l] = dh
        dW, db, dh = rgcn_bwd(blocks[l], g.R, ins[l], params[f"W{l}"], zs[l], relu=(l < L - 1),
                              dh_dst=dh, need_dh_src=(l > 0 or cfg.has_encoder))
        grads[f"W{l}"] = dW
        grads[f"b{l}"] = db
    extra = {"logits": logits, "dh": dhs, "ins": ins}
    if cfg.has_encoder:
        grads.update(encoder_bwd(g, params, blocks[0].src_gid, dh))
        extra["dH0"] = dh
    return StepResult(loss, blocks, x0, hs, zs, grads, extra)


def full_graph_infer(g: Graph, params: Dict[str, np.ndarray]) -> List[np.ndarray]:
    """Full-graph layer-wise inference (P:L393, P:L403 --inference /
    --save-embed-path): layer l maps every node's h_{l-1} (h_{-1} = input features) to h_l
    over its whole in-neighbourhood (fanout ALL, R-fanout ALL), i.e. the RGCN layer (R-rgcn)
    on one block whose dst and src lists are all nodes in gid order.  Returns [h_0 .. h_{L-1}],
    each (N_total, d) float64."""
    cfg = g.cfg
    L = len(cfg.fanouts)
    allg = np.arange(int(g.node_off[-1]), dtype=np.int64)
    blk = sample_blocks(g, allg, [-1], 0, 0)[0]
    assert np.array_equal(blk.src_gid, allg)          # every src is already a dst: no new nodes
    h = encoder_fwd(g, params, allg) if cfg.has_encoder else gather(g, allg).astype(np.float64)
    hs = []
    for l in range(L):
        _, h = rgcn_fwd(blk, g.R, h, params[f"W{l}"], params[f"b{l}"], relu=(l < L - 1))
        hs.append(h)
    return hs


def nc_predict(h: np.ndarray, Wc: np.ndarray, bc: np.ndarray):
    """Decoder logits (R-ncloss) and their argmax (lowest class on ties) and top-2 margin."""
    logits = np.asarray(h, np.float64) @ np.asarray(Wc, np.float64) + np.asarray(bc, np.float64)
    pred = np.argmax(logits, axis=1)
    top2 = np.sort(logits, axis=1)[:, -2:]
    return logits, pred, top2[:, 1] - top2[:, 0]


def lp_mrr(scores: np.ndarray):
    """MRR of link prediction (the paper's LP metric, Table 2, Table 6
    P:L249-259), reading R-mrr: row i of scores is [pos_i, neg_i1 .. neg_iK]; the positive's
    rank is 1 + #(negatives scoring higher) + #(negatives scoring equal) / 2 -- its expected
    rank under a uniformly random order of tied scores; MRR = mean over rows of 1 / rank.
    Returns (reciprocal ranks [B] float64, MRR)."""
    S = np.asarray(scores)
    B = S.shape[0]
    rr = np.zeros(B)
    for i in range(B):
        pos = S[i, 0]
        greater = 0
        equal = 0
        for x in S[i, 1:]:
            if x > pos:
                greater += 1
            elif x == pos:
                equal += 1
        rr[i] = 1.0 / (1.0 + greater + 0.5 * equal)
    return rr, (float(rr.mean()) if B else 0.0)


def lp_seeds(u: np.ndarray, v: np.ndarray, neg: np.ndarray) -> np.ndarray:
    """LP seed set (§8(a) a9): S0 = ascending unique(u ∪ v ∪ neg)."""
    return np.unique(np.concatenate([u, v, neg]).astype(np.int64))


def lp_step(g: Graph, params: Dict[str, np.ndarray], u: np.ndarray, v: np.ndarray, step: int,
            rng_seed: int, loss_kind: int = 0, neg_sampler: str = "joint", score: str = "distmult",
            local_range=None, w=None, pos_base: int = 0, group_base: int = 0) -> StepResult:
    """One LP step (§8(a) a3', a9, a10) in the paper's order.  neg_sampler (App. A.2.1):
    joint / uniform / local_joint (joint draws over local_range = (first local id, count) of
    the dst type) / in_batch; score: distmult (Eq. 3) or dot (Eq. 2); loss_kind 2 uses the
    per-positive weights w (Eq. 5)."""
    cfg = g.cfg
    L = len(cfg.fanouts)
    et = cfg.etypes[cfg.lp_etype]
    B = len(u)
    K = cfg.num_neg
    base, n_dst = int(g.node_off[et.dst]), int(cfg.counts[et.dst])
    if neg_sampler == "joint":
        neg = joint_negatives(B, K, n_dst, base, rng_seed, step, group_base)
        mode, group = 0, K
    elif neg_sampler == "local_joint":
        lo, cnt = local_range if local_range is not None else (0, n_dst)
        neg = joint_negatives(B, K, cnt, base + lo, rng_seed, step, group_base)
        mode, group = 0, K
    elif neg_sampler == "uniform":
        neg = uniform_negatives(B, K, n_dst, base, rng_seed, step, pos_base)
        mode, group = 0, 1
    elif neg_sampler == "in_batch":
        neg = np.zeros(0, np.int64)
        K = B - 1
        mode, group = 1, 1
    else:
        raise ValueError(neg_sampler)
    seeds = lp_seeds(u, v, neg)
    blocks = sample_blocks(g, seeds, cfg.fanouts, rng_seed, step, u, v, cfg.lp_etype, cfg.lp_rev_etype)
    x0 = gather(g, blocks[0].src_gid)
    h = x0.astype(np.float64)
    hs, zs, ins = [], [], []
    for l in range(L):
        ins.append(h)
        z, h = rgcn_fwd(blocks[l], g.R, h, params[f"W{l}"], params[f"b{l}"], relu=(l < L - 1))
        zs.append(z)
        hs.append(h)
    iu = np.searchsorted(seeds, u)
    iv = np.searchsorted(seeds, v)
    ineg = np.searchsorted(seeds, neg)
    rel = params["rel"] if score == "distmult" else None
    loss, scores, dhu, dhv, dhn, drel = lp_loss_ex(h[iu], h[iv], h[ineg] if mode == 0 else None, rel, K, group,
                                                   mode, loss_kind, w)
    dh = np.zeros_like(h)
    np.add.at(dh, iu, dhu)
    np.add.at(dh, iv, dhv)
    if mode == 0:
        np.add.at(dh, ineg, dhn)
    grads = {"rel": drel} if rel is not None else {}
    dhs = [None] * L
    for l in reversed(range(L)):
        dhs[l] = dh
        dW, db, dh = rgcn_bwd(blocks[l], g.R, ins[l], params[f"W{l}"], zs[l], relu=(l < L - 1),
                              dh_dst=dh, need_dh_src=(l > 0))
        grads[f"W{l}"] = dW
        grads[f"b{l}"] = db
    return StepResult(loss, blocks, x0, hs, zs, grads, {"neg": neg, "seeds": seeds, "scores": scores, "dh": dhs,
                                                        "ins": ins})


def train_step(g: Graph, params: Dict[str, np.ndarray], opt: Dict[str, Dict[str, np.ndarray]], t: int,
               batch, step: int, rng_seed: int, lr: float) -> StepResult:
    """Full step incl. Adam (t = 1-based step count).  params/opt hold float64 arrays."""
    cfg = g.cfg
    if cfg.task == "nc":
        seeds, labels = batch
        res = nc_step(g, params, seeds, labels, step, rng_seed)
    else:
        u, v = batch
        res = lp_step(g, params, u, v, step, rng_seed)
    for k, gr in res.grads.items():
        adam(params[k], gr, opt[k]["m"], opt[k]["v"], lr, t)
    return res
