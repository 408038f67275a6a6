"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module is the ONLY code both sides use.  It holds
none of the method's arithmetic: no sampling, no RNG the method draws, no layer,
loss or optimizer math.  It only defines *inputs*:

  * heterograph schemas shaped like the paper's workloads
    (BASELINE.json configs),
  * COO edge lists with a power-law degree profile (Chung-Lu style, weight of node
    rank k ~ (k+1)^-2/3, i.e. degree exponent ~2.5; SURVEY.md §8(d) "est." note),
  * node features uniform in [-1, 1), labels uniform in [0, C), train splits,
  * Glorot-uniform initial weights (SPEC S:L439 design decision).

Every value is a pure function of (seed, stream, index) through a 32-bit integer
hash, so the numpy (host) and torch (device) generators produce bit-identical
values: large configs are generated on the device with torch ops, and the oracle
re-derives any row it needs on the host without a copy from the CUDA path.
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional, Sequence, Tuple

import numpy as np

M32 = 0xFFFFFFFF
GOLDEN = 0x9E3779B9


# --------------------------------------------------------------------------------------
# 32-bit integer hash (Wellons "lowbias32"), written with 16-bit split multiplies so the
# same code is exact in numpy uint64 and in torch int64 (no signed overflow anywhere).
# --------------------------------------------------------------------------------------
def _mul32(x, c: int):
    lo = c & 0xFFFF
    hi = c >> 16
    return (x * lo + (((x * hi) & 0xFFFF) << 16)) & M32


def _mix32(x):
    x = x ^ (x >> 16)
    x = _mul32(x, 0x7FEB352D)
    x = x ^ (x >> 15)
    x = _mul32(x, 0x846CA68B)
    x = x ^ (x >> 16)
    return x


def hash32(seed: int, stream: int, idx, sub: int = 0):
    """h(seed, stream, idx, sub) -> uint32 values (same dtype/backend as idx).

    idx: numpy uint64/int64 array or torch int64 tensor of non-negative values < 2^62.
    """
    h1 = _mix32_scalar((seed + stream * GOLDEN) & M32)
    h1 = _mix32_scalar(h1 ^ ((seed >> 32) & M32))
    lo = idx & M32
    hi = (idx >> 32) & M32
    h2 = _mix32(lo ^ h1)
    h3 = _mix32(h2 ^ ((hi + sub * 0x85EBCA6B) & M32))
    return h3


def _mix32_scalar(x: int) -> int:
    return int(_mix32(np.uint64(x)))


# --------------------------------------------------------------------------------------
# Schemas
# --------------------------------------------------------------------------------------
@dataclasses.dataclass
class EType:
    name: str
    src: int
    dst: int
    num_edges: int
    reverse_of: Optional[int] = None  # etype id whose (src,dst) pairs this one reverses


@dataclasses.dataclass
class Config:
    name: str
    ntypes: List[str]
    counts: List[int]
    etypes: List[EType]
    feat_dim: int
    fanouts: List[int]          # f[l] for GNN layer l (layer 0 = input layer), SURVEY §8(c).4
    batch: int
    hidden: int
    num_classes: int
    target_ntype: int
    task: str = "nc"            # "nc" | "lp"
    lp_etype: int = -1          # LP target etype
    lp_rev_etype: int = -1      # its reverse etype (excluded too)
    num_neg: int = 32           # K for joint negative sampling
    train_frac: float = 0.8     # Fig. 6 split_pct [0.8, 0.1, 0.1]
    gen_seed: int = 2406060220
    rng_seed: int = 1           # the sampler's Philox key (method RNG input)
    lr: float = 1e-3
    feat_dtype: str = "f32"     # "f32" | "bf16": storage type of the node features (c.8)
    # input encoder (§8(a) a6): per-ntype raw feature width (None = feat_dim for
    # all) and which ntypes get a trainable projection Win{t} (dims[t] -> feat_dim); the
    # others are frozen tables of width feat_dim (featureless ntypes)
    feat_dims: Optional[List[int]] = None
    project: Optional[List[bool]] = None

    @property
    def num_ntypes(self) -> int:
        return len(self.ntypes)

    @property
    def num_etypes(self) -> int:
        return len(self.etypes)

    @property
    def node_off(self) -> np.ndarray:
        return np.concatenate([[0], np.cumsum(np.asarray(self.counts, dtype=np.int64))]).astype(np.int64)

    @property
    def num_nodes(self) -> int:
        return int(sum(self.counts))

    @property
    def num_edges(self) -> int:
        return int(sum(e.num_edges for e in self.etypes))

    def dim_of(self, t: int) -> int:
        """Raw feature width of ntype t."""
        return self.feat_dims[t] if self.feat_dims else self.feat_dim

    @property
    def has_encoder(self) -> bool:
        return bool(self.project) and any(self.project)

    @property
    def feat_seed(self) -> int:
        return self.gen_seed ^ 0xF

    def etype_src(self) -> np.ndarray:
        return np.array([e.src for e in self.etypes], dtype=np.int32)

    def etype_dst(self) -> np.ndarray:
        return np.array([e.dst for e in self.etypes], dtype=np.int32)


def tiny() -> Config:
    """configs[0]: 3 ntypes, 4 etypes, 10k nodes, 100k edges, 64-d, [5,5], b256, NC (C=8)."""
    return Config(
        name="tiny", ntypes=["A", "B", "C"], counts=[5000, 3000, 2000],
        etypes=[EType("r0", 0, 0, 40000), EType("r1", 0, 1, 15000),
                EType("r2", 1, 2, 20000), EType("r3", 2, 0, 25000)],
        feat_dim=64, fanouts=[5, 5], batch=256, hidden=128, num_classes=8,
        target_ntype=0, gen_seed=2406060220 + 1)


def mag() -> Config:
    """configs[1]: ogbn-mag-shaped (OGB counts, SURVEY §8(d) cfg 2), 128-d, [15,10], b1024.

    Reading (DESIGN.md R-cfg2): 21.1M forward edges + 3 reverse etypes = 36.8M stored,
    so that every ntype receives messages.
    """
    et = [EType("writes", 1, 0, 7145660), EType("cites", 0, 0, 5416271),
          EType("has_topic", 0, 3, 7505078), EType("affiliated_with", 1, 2, 1043998)]
    et += [EType("rev_writes", 0, 1, 7145660, reverse_of=0),
           EType("rev_has_topic", 3, 0, 7505078, reverse_of=2),
           EType("rev_affiliated_with", 2, 1, 1043998, reverse_of=3)]
    return Config(
        name="mag", ntypes=["paper", "author", "institution", "field"],
        counts=[736389, 1134649, 8740, 59965], etypes=et, feat_dim=128,
        fanouts=[15, 10], batch=1024, hidden=128, num_classes=349, target_ntype=0,
        gen_seed=2406060220 + 2)


def amazon_lp(scale: float = 1.0 / 8) -> Config:
    """configs[2]: Amazon-review-shaped LP, joint K=32, B=4096."""
    c = [int(10_000_000 * scale), int(232_967_461 * scale), int(43_494_913 * scale)]
    et = [EType("also_buy", 0, 0, int(355_037_927 * scale)),
          EType("receives", 0, 1, int(232_967_461 * scale)),
          EType("rev_receives", 1, 0, int(232_967_461 * scale), reverse_of=1),
          EType("writes", 2, 1, int(232_967_461 * scale))]
    return Config(
        name="amazon_lp", ntypes=["item", "review", "customer"], counts=c, etypes=et,
        feat_dim=128, fanouts=[10, 10], batch=4096, hidden=128, num_classes=0,
        target_ntype=0, task="lp", lp_etype=0, lp_rev_etype=-1, num_neg=32,
        gen_seed=2406060220 + 3)


def tiny_lp() -> Config:
    """Small LP case for parity: tiny graph, LP on r0 (A->A) with a reverse etype r4."""
    cfg = tiny()
    cfg.name = "tiny_lp"
    cfg.etypes = cfg.etypes + [EType("r0_rev", 0, 0, 40000, reverse_of=0)]
    cfg.task = "lp"
    cfg.lp_etype = 0
    cfg.lp_rev_etype = 4
    cfg.batch = 256
    cfg.num_neg = 16
    cfg.num_classes = 0
    cfg.gen_seed = 2406060220 + 11
    return cfg


def synth_1b(scale: float = 1.0) -> Config:
    """configs[4]: Table-3-shaped power-law heterograph: avg degree 100, 64-d."""
    n = [int(6_000_000 * scale), int(2_500_000 * scale), int(1_500_000 * scale)]
    E = int(1_000_000_000 * scale)
    et = [EType("r0", 0, 0, int(0.40 * E)), EType("r1", 0, 1, int(0.15 * E)),
          EType("r2", 1, 2, int(0.20 * E)), EType("r3", 2, 0, int(0.25 * E))]
    return Config(
        name="synth_1b", ntypes=["A", "B", "C"], counts=n, etypes=et, feat_dim=64,
        fanouts=[10, 10], batch=1024, hidden=128, num_classes=16, target_ntype=0,
        gen_seed=2406060220 + 5)


def gcn_1b(scale: float = 1.0) -> Config:
    """Table 3: homogeneous synthetic graph with 1B edges, average degree 100
    (10M nodes), 64-d features, a GCN for node classification with 80 % training nodes (8M, as
    the table's caption states).  GCN = the RGCN layer with one relation (R-gcn): mean over the
    sampled in-neighbours + self loop.  Fanouts / batch / classes as configs[4]."""
    n = int(10_000_000 * scale)
    return Config(
        name="gcn_1b" if scale == 1.0 else f"gcn_1b_x{scale:g}", ntypes=["node"], counts=[n],
        etypes=[EType("edge", 0, 0, int(1_000_000_000 * scale))], feat_dim=64, fanouts=[10, 10], batch=1024,
        hidden=128, num_classes=16, target_ntype=0, gen_seed=2406060220 + 6)


def mag240m(scale: float = 1.0) -> Config:
    """configs[3]: MAG240M-shaped (OGB-LSC counts [EXT], SURVEY §8(d) cfg 4): paper 768-d bf16
    features with a trainable input projection 768 -> 128 (a6); author / institution are
    featureless -> frozen 128-d bf16 tables; 3 forward + 2 reverse etypes
    (2.16B stored at full scale), [15,10], b1024/GPU, NC on paper, C = 153."""
    c = [int(121_751_666 * scale), int(122_383_112 * scale), int(25_721 * scale)]
    et = [EType("writes", 1, 0, int(386_022_720 * scale)), EType("cites", 0, 0, int(1_297_748_926 * scale)),
          EType("affiliated_with", 1, 2, int(44_592_586 * scale))]
    et += [EType("rev_writes", 0, 1, int(386_022_720 * scale), reverse_of=0),
           EType("rev_affiliated_with", 2, 1, int(44_592_586 * scale), reverse_of=2)]
    return Config(
        name="mag240m" if scale == 1.0 else f"mag240m_x{scale:g}", ntypes=["paper", "author", "institution"],
        counts=c, etypes=et, feat_dim=128, fanouts=[15, 10], batch=1024, hidden=128, num_classes=153,
        target_ntype=0, gen_seed=2406060220 + 4, feat_dtype="bf16", feat_dims=[768, 128, 128],
        project=[True, False, False])


def tiny_enc() -> Config:
    """Small input-encoder case for parity: tiny graph, ntype A with 256-d raw features and a
    projection to 128, B / C frozen 128-d tables (bf16 storage)."""
    cfg = tiny()
    cfg.name = "tiny_enc"
    cfg.feat_dtype = "bf16"
    cfg.feat_dim = 128
    cfg.feat_dims = [256, 128, 128]
    cfg.project = [True, False, False]
    cfg.gen_seed = 2406060220 + 12
    return cfg


def with_dtype(cfg: Config, feat_dtype: str) -> Config:
    """The same workload with features stored as `feat_dtype` ("f32" | "bf16")."""
    if feat_dtype == cfg.feat_dtype:
        return cfg
    return dataclasses.replace(cfg, feat_dtype=feat_dtype, name=f"{cfg.name}_{feat_dtype}")


CONFIGS = {"tiny": tiny, "mag": mag, "amazon_lp": amazon_lp, "tiny_lp": tiny_lp,
           "synth_1b": synth_1b, "mag240m": mag240m, "mag240m_1_16": lambda: mag240m(1.0 / 16),
           "tiny_enc": tiny_enc, "gcn_1b": gcn_1b, "synth_10b": lambda: synth_1b(10.0)}


def get(name: str) -> Config:
    return CONFIGS[name]()


def scaled(cfg: Config, s: float, name: Optional[str] = None) -> Config:
    """Same schema with node and edge counts scaled by s (parity cases at small size)."""
    c = dataclasses.replace(cfg)
    c.counts = [max(2, int(n * s)) for n in cfg.counts]
    c.etypes = [dataclasses.replace(e, num_edges=max(1, int(e.num_edges * s))) for e in cfg.etypes]
    for i, e in enumerate(c.etypes):
        if e.reverse_of is not None:
            e.num_edges = c.etypes[e.reverse_of].num_edges
    c.name = name or f"{cfg.name}_x{s:g}"
    return c


# --------------------------------------------------------------------------------------
# Edges: per etype COO (local ids, int32).  Rank r = floor(N * x^3) with x uniform gives
# P(rank) ~ (rank+1)^(-2/3) (continuous Chung-Lu weights).  Ranks are mapped to ids by an
# affine bijection id = (a*rank + b) mod N so hubs are scattered over the id space.
# --------------------------------------------------------------------------------------
_PRIMES = [2654435761, 2246822519, 3266489917, 668265263, 374761393, 1103515245 | 1,
           4294967291, 2147483647, 1000000007, 998244353]


def _affine(n: int, t: int) -> Tuple[int, int]:
    for p in _PRIMES[t % len(_PRIMES):] + _PRIMES:
        if n % p != 0 and p % n != 0:
            return p % n if p % n != 0 else 1, (t * 7919) % n
    return 1, 0


def _endpoint_ids(seed: int, stream: int, n: int, t: int, idx, backend):
    h = hash32(seed, stream, idx)
    if backend == "np":
        x = h.astype(np.float64) * (1.0 / 4294967296.0)
        rank = np.floor(float(n) * (x * x * x)).astype(np.int64)
        rank = np.minimum(rank, n - 1)
    else:
        import torch
        x = h.to(torch.float64) * (1.0 / 4294967296.0)
        rank = torch.floor(float(n) * (x * x * x)).to(torch.int64)
        rank = torch.clamp(rank, max=n - 1)
    a, b = _affine(n, t)
    return (rank * a + b) % n


def etype_coo(cfg: Config, r: int, backend: str = "np", device=None, lo: int = 0, hi: Optional[int] = None):
    """COO (src_local, dst_local) int32 of etype r, edges [lo, hi) in generation order."""
    e = cfg.etypes[r]
    base = r if e.reverse_of is None else e.reverse_of
    be = cfg.etypes[base]
    hi = be.num_edges if hi is None else hi
    if backend == "np":
        idx = np.arange(lo, hi, dtype=np.uint64)
    else:
        import torch
        idx = torch.arange(lo, hi, dtype=torch.int64, device=device)
    s = _endpoint_ids(cfg.gen_seed, 2 * base, cfg.counts[be.src], be.src, idx, backend)
    d = _endpoint_ids(cfg.gen_seed, 2 * base + 1, cfg.counts[be.dst], be.dst + 17, idx, backend)
    if e.reverse_of is not None:
        s, d = d, s
    if backend == "np":
        return s.astype(np.int32), d.astype(np.int32)
    import torch
    return s.to(torch.int32), d.to(torch.int32)


# --------------------------------------------------------------------------------------
# Features, labels, splits
# --------------------------------------------------------------------------------------
def _round_bf16_bits(bits):
    """fp32 bit patterns -> nearest-even bf16 bit patterns (kept in the high 16 bits).
    Integer-only so numpy and torch give identical values (finite inputs)."""
    return (bits + 0x7FFF + ((bits >> 16) & 1)) & 0xFFFF0000


def feature_rows(cfg: Config, t: int, local_ids, backend: str = "np", device=None):
    """F_t[i, k] = (h >> 8) * 2^-23 - 1, exactly representable in fp32, in [-1, 1).  With
    cfg.feat_dtype == "bf16" each value is rounded to the nearest bf16 (ties to even), so the
    returned fp32 values are exactly representable in bf16."""
    d = cfg.dim_of(t)
    bf = cfg.feat_dtype == "bf16"
    if backend == "np":
        ids = np.asarray(local_ids, dtype=np.uint64)
        idx = ids[:, None] * np.uint64(d) + np.arange(d, dtype=np.uint64)[None, :]
        h = hash32(cfg.feat_seed, 1000 + t, idx)
        f = ((h >> 8).astype(np.float32) * np.float32(2.0 ** -23) - np.float32(1.0)).astype(np.float32)
        if bf:
            b = f.view(np.uint32).astype(np.uint64)
            f = (_round_bf16_bits(b) & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.float32)
        return f
    import torch
    ids = torch.as_tensor(local_ids, dtype=torch.int64, device=device)
    idx = ids[:, None] * d + torch.arange(d, dtype=torch.int64, device=device)[None, :]
    h = hash32(cfg.feat_seed, 1000 + t, idx)
    f = (h >> 8).to(torch.float32) * (2.0 ** -23) - 1.0
    if bf:
        b = f.view(torch.int32).to(torch.int64) & 0xFFFFFFFF
        f = (_round_bf16_bits(b) & 0xFFFFFFFF).to(torch.int64)
        f = torch.where(f >= 2 ** 31, f - 2 ** 32, f).to(torch.int32).view(torch.float32)
    return f


def feature_table(cfg: Config, t: int, backend: str = "np", device=None, chunk: Optional[int] = None,
                  lo: int = 0, hi: Optional[int] = None):
    """Rows [lo, hi) (default: all) of ntype t's table: numpy float32 (values exact in the
    config's dtype), or a torch tensor of the config's storage dtype (float32 / bfloat16;
    the conversion is exact)."""
    hi = cfg.counts[t] if hi is None else hi
    n = hi - lo
    d = cfg.dim_of(t)
    chunk = chunk or max(1, (1 << 26) // d)          # ~64M elements per generation chunk
    if backend == "np":
        out = np.empty((n, d), dtype=np.float32)
        for a in range(lo, hi, chunk):
            b = min(hi, a + chunk)
            out[a - lo:b - lo] = feature_rows(cfg, t, np.arange(a, b), "np")
        return out
    import torch
    dt = torch.bfloat16 if cfg.feat_dtype == "bf16" else torch.float32
    out = torch.empty((n, d), dtype=dt, device=device)
    for a in range(lo, hi, chunk):
        b = min(hi, a + chunk)
        out[a - lo:b - lo] = feature_rows(cfg, t, torch.arange(a, b, device=device), "torch", device).to(dt)
    return out


def labels(cfg: Config, backend: str = "np", device=None):
    t = cfg.target_ntype
    n = cfg.counts[t]
    C = max(cfg.num_classes, 1)
    if backend == "np":
        h = hash32(cfg.gen_seed, 2000 + t, np.arange(n, dtype=np.uint64))
        return (h % np.uint64(C)).astype(np.int32)
    import torch
    h = hash32(cfg.gen_seed, 2000 + t, torch.arange(n, dtype=torch.int64, device=device))
    return (h % C).to(torch.int32)


def train_nodes(cfg: Config) -> np.ndarray:
    """Local ids of target-type training nodes (split_pct 0.8, Fig. 6)."""
    n = cfg.counts[cfg.target_ntype]
    h = hash32(cfg.gen_seed, 3000, np.arange(n, dtype=np.uint64))
    return np.nonzero((h % np.uint64(1000)) < np.uint64(int(cfg.train_frac * 1000)))[0].astype(np.int64)


_PERM_CACHE = {}


def epoch_perm(n: int, epoch: int, seed: int) -> np.ndarray:
    key = (n, epoch, seed)
    if key not in _PERM_CACHE:
        if len(_PERM_CACHE) > 8:
            _PERM_CACHE.clear()
        _PERM_CACHE[key] = np.random.Generator(np.random.PCG64([seed, epoch])).permutation(n)
    return _PERM_CACHE[key]


def nc_seeds(cfg: Config, step: int, train: Optional[np.ndarray] = None) -> np.ndarray:
    """Seed batching (§8(a) a1): batch = consecutive slice of an epoch permutation; gids."""
    if train is None:
        train = train_nodes(cfg)
    B = cfg.batch
    per_epoch = max(1, len(train) // B)
    ep, k = divmod(step, per_epoch)
    perm = epoch_perm(len(train), ep, cfg.gen_seed)
    loc = train[perm[k * B:(k + 1) * B]]
    return (loc + cfg.node_off[cfg.target_ntype]).astype(np.int64)


def lp_train_edges(cfg: Config, step: int) -> Tuple[np.ndarray, np.ndarray]:
    """LP batch (§8(a) a1): B positive (u, v) gids of the target etype, edge index slice of an
    epoch permutation over the training edges (first 80% by hash split)."""
    e = cfg.etypes[cfg.lp_etype]
    E = e.num_edges
    h = hash32(cfg.gen_seed, 4000, np.arange(E, dtype=np.uint64))
    tr = np.nonzero((h % np.uint64(1000)) < np.uint64(int(cfg.train_frac * 1000)))[0]
    B = cfg.batch
    per_epoch = max(1, len(tr) // B)
    ep, k = divmod(step, per_epoch)
    perm = epoch_perm(len(tr), ep, cfg.gen_seed + 1)
    ids = tr[perm[k * B:(k + 1) * B]]
    s, d = etype_coo(cfg, cfg.lp_etype)
    off = cfg.node_off
    return (s[ids].astype(np.int64) + off[e.src], d[ids].astype(np.int64) + off[e.dst])


class LPBatcher:
    """Cached LP batch source (same batches as lp_train_edges, without regenerating the COO)."""

    def __init__(self, cfg: Config):
        self.cfg = cfg
        e = cfg.etypes[cfg.lp_etype]
        h = hash32(cfg.gen_seed, 4000, np.arange(e.num_edges, dtype=np.uint64))
        self.tr = np.nonzero((h % np.uint64(1000)) < np.uint64(int(cfg.train_frac * 1000)))[0]
        self.s, self.d = etype_coo(cfg, cfg.lp_etype)
        self.off = cfg.node_off
        self.e = e
        self._perm = {}

    def batch(self, step: int):
        B = self.cfg.batch
        per_epoch = max(1, len(self.tr) // B)
        ep, k = divmod(step, per_epoch)
        if ep not in self._perm:
            self._perm = {ep: epoch_perm(len(self.tr), ep, self.cfg.gen_seed + 1)}
        ids = self.tr[self._perm[ep][k * B:(k + 1) * B]]
        return (self.s[ids].astype(np.int64) + self.off[self.e.src], self.d[ids].astype(np.int64) + self.off[self.e.dst])


def lp_keep_mask(cfg: Config) -> np.ndarray:
    """Val/test LP edges are removed from the training graph: keep = train split."""
    e = cfg.etypes[cfg.lp_etype]
    h = hash32(cfg.gen_seed, 4000, np.arange(e.num_edges, dtype=np.uint64))
    return (h % np.uint64(1000)) < np.uint64(int(cfg.train_frac * 1000))


# --------------------------------------------------------------------------------------
# Initial parameters (inputs, not method arithmetic)
# --------------------------------------------------------------------------------------
def glorot(shape: Sequence[int], fan_in: int, fan_out: int, seed: int) -> np.ndarray:
    a = np.sqrt(6.0 / (fan_in + fan_out))
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.uniform(-a, a, size=shape).astype(np.float32)


def init_params(cfg: Config) -> dict:
    """RGCN params per layer l: W[l] (R+1, d_in, d_out) with slot R = W_self; b[l] (d_out,).
    NC decoder Wc (hidden, C), bc (C,); LP relation embedding rel (hidden,)."""
    L = len(cfg.fanouts)
    R = cfg.num_etypes
    p = {}
    for t in range(cfg.num_ntypes):   # input encoder projections (a6)
        if cfg.project and cfg.project[t]:
            p[f"Win{t}"] = glorot((cfg.dim_of(t), cfg.feat_dim), cfg.dim_of(t), cfg.feat_dim, cfg.gen_seed * 31 + 50 + t)
    d_in = cfg.feat_dim
    for l in range(L):
        d_out = cfg.hidden
        p[f"W{l}"] = glorot((R + 1, d_in, d_out), d_in, d_out, cfg.gen_seed * 31 + l)
        p[f"b{l}"] = np.zeros(d_out, dtype=np.float32)
        d_in = d_out
    if cfg.task == "nc":
        p["Wc"] = glorot((cfg.hidden, cfg.num_classes), cfg.hidden, cfg.num_classes, cfg.gen_seed * 31 + 99)
        p["bc"] = np.zeros(cfg.num_classes, dtype=np.float32)
    else:
        p["rel"] = np.random.Generator(np.random.PCG64(cfg.gen_seed * 31 + 98)).uniform(
            -1.0, 1.0, size=cfg.hidden).astype(np.float32)
    return p


def param_order(cfg: Config) -> List[str]:
    L = len(cfg.fanouts)
    names = [f"Win{t}" for t in range(cfg.num_ntypes) if cfg.project and cfg.project[t]]
    for l in range(L):
        names += [f"W{l}", f"b{l}"]
    names += ["Wc", "bc"] if cfg.task == "nc" else ["rel"]
    return names
