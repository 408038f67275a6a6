"""Thin Python driver over libgsb: device memory (torch tensors), streams, and the order of
C-ABI calls that make one RGCN mini-batch train step (Fig. 4; Fig. 8
P:L480-489).  Every arithmetic step runs in libgsb's CUDA kernels; this module only
allocates buffers and passes pointers.
"""
from __future__ import annotations

import os
import ctypes as C
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import call, lib

# feature element types of the C ABI (GSB_F32 / GSB_BF16)
DTYPE_CODE = {torch.float32: 0, torch.bfloat16: 1}


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream: Optional[torch.cuda.Stream] = None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _require_cuda():
    if not torch.cuda.is_available():
        raise _lib.GsbError("libgsb needs a CUDA device (there is no CPU fallback)")


class _PeerTable:
    """Marker for a learnable table held by a dist.PeerEmbedding (partitioned over ranks)."""

    def __init__(self, pe):
        self.pe = pe


class GraphStore:
    """Per-etype CSC + per-ntype feature tables resident in HBM."""

    def __init__(self, counts: Sequence[int], etype_src: Sequence[int], etype_dst: Sequence[int],
                 device: str = "cuda"):
        _require_cuda()
        self.device = torch.device(device)
        self.counts = np.asarray(counts, dtype=np.int64)
        self.etype_src = np.asarray(etype_src, dtype=np.int32)
        self.etype_dst = np.asarray(etype_dst, dtype=np.int32)
        self.T, self.R = len(self.counts), len(self.etype_src)
        self.node_off = np.concatenate([[0], np.cumsum(self.counts)]).astype(np.int64)
        h = C.c_void_p()
        call("gsb_graph_create", self.T, self.counts.ctypes.data_as(C.c_void_p), self.R,
             self.etype_src.ctypes.data_as(C.c_void_p), self.etype_dst.ctypes.data_as(C.c_void_p), C.byref(h))
        self.h = h
        self.indptr: List[Optional[torch.Tensor]] = [None] * self.R
        self.indices: List[Optional[torch.Tensor]] = [None] * self.R
        self.n_edges = [0] * self.R
        self.feats: List[Optional[torch.Tensor]] = [None] * self.T
        self.feat_dim = 0
        self.feat_dtype = torch.float32

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().gsb_graph_destroy(self.h)
        except Exception:
            pass

    def construct_features(self, ntype: int, featured: Sequence[int], dim: int, first: int = 0,
                           count: Optional[int] = None, stream=None) -> torch.Tensor:
        """Eq. 1 (§8(f) f4): fp32 rows [first, first+count) of ntype built as the
        average of its featured in-neighbours' rows (gsb_construct_features)."""
        count = int(self.counts[ntype]) - first if count is None else count
        out = torch.empty((count, dim), dtype=torch.float32, device=self.device)
        mask = 0
        for t in featured:
            mask |= 1 << int(t)
        call("gsb_construct_features", self.h, ntype, mask, first, count, _ptr(out), dim, _stream(stream))
        return out

    def load_etype(self, r: int, src: torch.Tensor, dst: torch.Tensor, keep: Optional[torch.Tensor] = None):
        """gsb_csc_build from a device COO (int32 local ids)."""
        s = torch.as_tensor(src, dtype=torch.int32).to(self.device).contiguous()
        d = torch.as_tensor(dst, dtype=torch.int32).to(self.device).contiguous()
        k = None if keep is None else torch.as_tensor(keep, dtype=torch.uint8).to(self.device).contiguous()
        n = s.numel()
        ws_b = C.c_size_t()
        call("gsb_csc_build_bytes", self.h, r, n, C.byref(ws_b))
        ws = torch.empty(max(int(ws_b.value), 1), dtype=torch.uint8, device=self.device)
        n_dst = int(self.counts[self.etype_dst[r]])
        indptr = torch.empty(n_dst + 1, dtype=torch.int64, device=self.device)
        indices = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        kept = C.c_int64()
        call("gsb_csc_build", self.h, r, _ptr(s), _ptr(d), _ptr(k), n, _ptr(indptr), _ptr(indices), C.byref(kept),
             _ptr(ws), ws.numel(), _stream())
        del ws
        self.indptr[r] = indptr
        self.indices[r] = indices
        self.n_edges[r] = int(kept.value)

    def load_etype_range(self, r: int, src: torch.Tensor, dst: torch.Tensor, lo: int, hi: int,
                         keep: Optional[torch.Tensor] = None, eid_base: Optional[int] = None):
        """gsb_csc_build_range: this rank's shard of etype r's CSC -- the in-edges of the dst
        local ids [lo, hi) it owns (§8(e), node-ID partition); eid_base = global position of
        the shard's first edge (counted by the build over the given COO, or given by the caller
        when the COO passed is already restricted to the range)."""
        s = torch.as_tensor(src, dtype=torch.int32).to(self.device).contiguous()
        d = torch.as_tensor(dst, dtype=torch.int32).to(self.device).contiguous()
        k = None if keep is None else torch.as_tensor(keep, dtype=torch.uint8).to(self.device).contiguous()
        n = s.numel()
        ws_b = C.c_size_t()
        call("gsb_csc_build_bytes", self.h, r, n, C.byref(ws_b))
        ws = torch.empty(max(int(ws_b.value), 1), dtype=torch.uint8, device=self.device)
        indptr = torch.empty(hi - lo + 1, dtype=torch.int64, device=self.device)
        # capacity: every edge could fall in range; trimmed to the kept count below
        indices = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        kept, before = C.c_int64(), C.c_int64()
        call("gsb_csc_build_range", self.h, r, _ptr(s), _ptr(d), _ptr(k), n, lo, hi, _ptr(indptr), _ptr(indices),
             C.byref(kept), C.byref(before), _ptr(ws), ws.numel(), _stream())
        del ws
        indices = indices[:max(int(kept.value), 1)].clone()
        if eid_base is not None:
            before = C.c_int64(int(eid_base))
        call("gsb_graph_set_csc", self.h, r, _ptr(indptr), _ptr(indices), int(kept.value), int(before.value))
        self.indptr[r] = indptr
        self.indices[r] = indices
        self.n_edges[r] = int(kept.value)
        self.eid_base = getattr(self, "eid_base", [0] * self.R)
        self.eid_base[r] = int(before.value)
        self.part_range = getattr(self, "part_range", {})
        self.part_range[r] = (lo, hi)

    def set_features(self, t: int, feat: torch.Tensor):
        """Register ntype t's feature table (fp32 or bf16 rows; one format for all ntypes)."""
        dt = feat.dtype if feat.dtype in DTYPE_CODE else torch.float32
        f = feat.to(self.device, dtype=dt).contiguous()
        call("gsb_graph_set_features", self.h, t, _ptr(f), f.shape[1], DTYPE_CODE[dt])
        self.feats[t] = f
        self.feat_dim = f.shape[1]
        self.feat_dtype = dt

    def gather(self, gids: torch.Tensor) -> torch.Tensor:
        """gsb_gather: out[i] = F_{t(i)}[gid_i - off_t] (exact copy, feature dtype)."""
        g = gids.to(self.device, dtype=torch.int64).contiguous()
        out = torch.empty((g.numel(), self.feat_dim), dtype=self.feat_dtype, device=self.device)
        call("gsb_gather", self.h, _ptr(g), g.numel(), _ptr(out), _stream())
        return out

    def slot_etypes(self) -> List[List[int]]:
        res = []
        for t in range(self.T):
            lst = []
            for s in range(32):
                e = C.c_int32()
                call("gsb_slot_etype", self.h, t, s, C.byref(e))
                if e.value < 0:
                    break
                lst.append(e.value)
            res.append(lst)
        return res


@dataclass
class BlockArrays:
    dst_gid: torch.Tensor
    src_gid: torch.Tensor
    seg_ptr: torch.Tensor      # (n_dst * S + 1)
    e_src_gid: torch.Tensor
    e_eid: torch.Tensor
    e_src: torch.Tensor
    num_slots: int
    dst_type_cnt: np.ndarray
    src_type_cnt: np.ndarray


class MiniBatchSampler:
    """gsb_blocks_* : sampled message-flow blocks of one mini-batch in a device arena."""

    def __init__(self, store: GraphStore, fanouts: Sequence[int], max_seeds: int, max_excl: int = 0):
        self.max_excl = max_excl
        self.store = store
        self.L = len(fanouts)
        f = np.asarray(fanouts, dtype=np.int32)
        h = C.c_void_p()
        call("gsb_blocks_create", store.h, self.L, f.ctypes.data_as(C.c_void_p), max_seeds, max_excl, C.byref(h))
        self.h = h
        b = C.c_size_t()
        call("gsb_blocks_arena_bytes", self.h, C.byref(b))
        self.arena = torch.empty(int(b.value), dtype=torch.uint8, device=store.device)
        call("gsb_blocks_init_arena", self.h, _ptr(self.arena), self.arena.numel(), _stream())
        self.max_seeds = max_seeds
        self.fanouts = list(fanouts)

    def twin(self) -> "MiniBatchSampler":
        """A second sampler of the same shape (own handle + arena), for double buffering; a
        frontier exchange attached to this sampler (dist.SampleExchange) is attached to the twin
        too, with its own buffers."""
        tw = MiniBatchSampler(self.store, self.fanouts, self.max_seeds, self.max_excl)
        sx = getattr(self, "_sx", None)
        if sx is not None:
            from .dist import SampleExchange
            SampleExchange(tw, sx.world, sx.rank, first_hop=sx.first_hop, group=sx.group)
        return tw

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().gsb_blocks_destroy(self.h)
        except Exception:
            pass

    def sample(self, seeds: torch.Tensor, rng_seed: int, step: int, excl_u: Optional[torch.Tensor] = None,
               excl_v: Optional[torch.Tensor] = None, excl_etype: int = -1, excl_rev_etype: int = -1,
               stream=None, n_seeds_dev: Optional[torch.Tensor] = None, step_dev: Optional[torch.Tensor] = None,
               n_seeds: Optional[int] = None):
        """gsb_sample.  With n_seeds_dev the seed count is read on the device (n_seeds is then
        the capacity); with step_dev the RNG step word is read on the device."""
        a = _lib.gsb_sample_args()
        a.seeds = seeds.data_ptr()
        a.n_seeds = int(n_seeds if n_seeds is not None else seeds.numel())
        a.n_seeds_dev = None if n_seeds_dev is None else n_seeds_dev.data_ptr()
        a.rng_seed = rng_seed
        a.step = step
        a.step_dev = None if step_dev is None else step_dev.data_ptr()
        a.excl_u = None if excl_u is None else excl_u.data_ptr()
        a.excl_v = None if excl_v is None else excl_v.data_ptr()
        a.n_excl = 0 if excl_u is None else excl_u.numel()
        a.excl_etype = excl_etype
        a.excl_rev_etype = excl_rev_etype
        call("gsb_sample", self.h, C.byref(a), _ptr(self.arena), self.arena.numel(), _stream(stream))

    def input_gids(self):
        """(device view of the input-layer gids, their count) -- syncs to read the count."""
        nd, ns, ne = C.c_int64(), C.c_int64(), C.c_int64()
        call("gsb_block_sizes", self.h, _ptr(self.arena), 0, C.byref(nd), C.byref(ns), C.byref(ne), None, None,
             _stream())
        v = _lib.gsb_block_view()
        call("gsb_block_view_get", self.h, _ptr(self.arena), 0, C.byref(v))
        off = v.src_gid - self.arena.data_ptr()
        n = int(ns.value)
        return self.arena[off:off + max(n, 1) * 8].view(torch.int64), n

    def input_rows(self) -> int:
        v = C.c_int64()
        call("gsb_blocks_input_rows", self.h, C.byref(v))
        return int(v.value)

    def dst_rows(self, layer: int) -> int:
        v = C.c_int64()
        call("gsb_blocks_dst_rows", self.h, layer, C.byref(v))
        return int(v.value)

    def acat_floats(self, layer: int, d_in: int) -> int:
        v = C.c_int64()
        call("gsb_layer_acat_floats", self.h, layer, d_in, C.byref(v))
        return int(v.value)

    def poll_error(self) -> int:
        code = C.c_int32()
        st = lib().gsb_blocks_poll_error(self.h, _ptr(self.arena), C.byref(code), _stream())
        if st not in (0, 4):
            _lib.check(st, "gsb_blocks_poll_error")
        return int(code.value)

    def block(self, layer: int) -> BlockArrays:
        """Copy-free views of the block of `layer` (syncs to read the sizes)."""
        T = self.store.T
        nd, ns, ne = C.c_int64(), C.c_int64(), C.c_int64()
        dtc = np.zeros(T, np.int64)
        stc = np.zeros(T, np.int64)
        call("gsb_block_sizes", self.h, _ptr(self.arena), layer, C.byref(nd), C.byref(ns), C.byref(ne),
             dtc.ctypes.data_as(C.c_void_p), stc.ctypes.data_as(C.c_void_p), _stream())
        v = _lib.gsb_block_view()
        call("gsb_block_view_get", self.h, _ptr(self.arena), layer, C.byref(v))
        dev = self.store.device

        def view(ptr, n, dtype):
            if n == 0:
                return torch.empty(0, dtype=dtype, device=dev)
            return _from_ptr(ptr, n, dtype, dev, self.arena)

        S = v.num_slots
        return BlockArrays(view(v.dst_gid, nd.value, torch.int64), view(v.src_gid, ns.value, torch.int64),
                           view(v.seg_ptr, nd.value * S + 1, torch.int64), view(v.e_src_gid, ne.value, torch.int64),
                           view(v.e_eid, ne.value, torch.int64), view(v.e_src, ne.value, torch.int32), S, dtc, stc)


def _from_ptr(ptr: int, n: int, dtype: torch.dtype, device, owner: torch.Tensor) -> torch.Tensor:
    """A tensor view of n elements at device address ptr inside `owner`'s storage."""
    base = owner.data_ptr()
    esz = torch.empty(0, dtype=dtype).element_size()
    off = ptr - base
    assert off % esz == 0 and 0 <= off and off + n * esz <= owner.numel()
    return owner[off:off + n * esz].view(dtype).clone()


class _TrainerBase:
    """Shared state of an RGCN train step through libgsb: flat parameter / gradient / Adam
    buffers, upper-bound-sized activation buffers, device step counters (so a whole step can
    be captured in a CUDA graph and replayed), and the RGCN layers (§8(a) a5, a7, a11, a12)."""

    def __init__(self, store: GraphStore, fanouts: Sequence[int], max_seeds: int, hidden: int,
                 params: Dict[str, np.ndarray], param_order: Sequence[str], lr: float, rng_seed: int,
                 max_excl: int = 0):
        self.store = store
        self.L = len(fanouts)
        self.hidden = hidden
        self.lr = lr
        self.rng_seed = rng_seed
        self.sampler = MiniBatchSampler(store, fanouts, max_seeds=max_seeds, max_excl=max_excl)
        dev = store.device
        self.device = dev
        self.names = list(param_order)
        sizes = [int(np.prod(params[k].shape)) for k in self.names]
        self.offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        self.n_params = int(self.offsets[-1])
        self.flat = torch.from_numpy(np.concatenate([params[k].reshape(-1) for k in self.names])).to(dev)
        self.grad = torch.zeros_like(self.flat)
        self.m = torch.zeros_like(self.flat)
        self.v = torch.zeros_like(self.flat)
        self.shapes = {k: params[k].shape for k in self.names}
        self.t = 0
        d0 = int(params["W0"].shape[1])      # layer-0 input width (= encoder output width)
        self.d_in = [d0] + [hidden] * (self.L - 1)
        # input encoder (a6): ntypes with a projection Win{t}; the others are frozen tables
        # unless set_embedding() makes them learnable (f1)
        self.enc_types = [t for t in range(store.T) if f"Win{t}" in self.names]
        self.emb: Dict[int, tuple] = {}
        nin = self.sampler.input_rows()
        self.x0 = torch.empty((0 if self.enc_types else nin, d0), dtype=store.feat_dtype, device=dev)
        self.xperm = torch.empty(max(nin, 1), dtype=torch.int32, device=dev)   # C4/C5 bucketing permutation
        if self.enc_types:
            self.H0 = torch.empty((nin, d0), dtype=torch.float32, device=dev)
            self.dH0 = torch.empty((nin, d0), dtype=torch.float32, device=dev)
            self._win = (C.c_void_p * store.T)(*[self._pp(f"Win{t}").value if t in self.enc_types else None
                                                  for t in range(store.T)])
            self._dwin = (C.c_void_p * store.T)(*[self._pp(f"Win{t}", "g").value if t in self.enc_types else None
                                                   for t in range(store.T)])
            wb = C.c_size_t()
            call("gsb_encoder_ws_bytes", self.sampler.h, self._win, d0, C.byref(wb))
            self.enc_ws = torch.empty(max(int(wb.value), 1), dtype=torch.uint8, device=dev)
        self.hout = [torch.empty((self.sampler.dst_rows(l), hidden), dtype=torch.float32, device=dev)
                     for l in range(self.L)]
        self.acat = [torch.empty(self.sampler.acat_floats(l, self.d_in[l]), dtype=torch.float32, device=dev)
                     for l in range(self.L)]
        self.acat0 = self.acat[0]      # per-batch (double-buffered with the pipeline)
        self.early_agg = os.environ.get("GSB_EARLY_AGG", "1") != "0"   # A/B knob (NC)
        self.dacat = torch.empty(max(self.sampler.acat_floats(l, self.d_in[l]) for l in range(self.L)),
                                 dtype=torch.float32, device=dev)
        self.dh = [torch.empty((self.sampler.dst_rows(l), hidden), dtype=torch.float32, device=dev)
                   for l in range(self.L)]
        self.loss = torch.zeros(1, dtype=torch.float32, device=dev)
        # device counters: [0] = RNG step word, [1] = Adam t (graph mode)
        self.counters = torch.zeros(2, dtype=torch.int32, device=dev)
        self.graph = None
        self.graph_ws = 1
        self.graph_allreduce = None
        self.fuse_gather = True
        self.exchange = None      # dist.FeatureExchange when features are partitioned across GPUs
        self._bufs = None         # double-buffered per-batch state (enable_prefetch)
        self.pipe_graphs = None
        self.pipe_k = 0
        self._wimg_names = []
        self.flat_hi = self.flat_lo = None
        # pre-split layer weights for the TMA GEMMs (default; GSB_WIMG=0 off, =1 the separate
        # per-step refresh launch instead of Adam's fused split, profiles/round2_gemm_tma3.md)
        wimg = os.environ.get("GSB_WIMG", "adam")
        if wimg == "1":
            self._register_weight_images()
        elif wimg == "adam":
            self._register_weight_images_adam()

    def _register_weight_images(self):
        """tf32 hi/lo images of the layer weights (gsb_weight_images_*): the NN / NT GEMMs then
        TMA the split B operand instead of splitting W in every CTA; refreshed at the start of
        every compute phase (after the previous step's Adam).  The NC decoder weight is left
        out: its class-count row stride is not TMA-addressable (the GEMMs take the cp.async
        kernel there)."""
        self._wimg_names = [f"W{l}" for l in range(self.L)]
        self._wimg_bufs = []
        for name in self._wimg_names:
            shp = self.shapes[name]
            slots, K, N = (int(shp[0]), int(shp[1]), int(shp[2])) if len(shp) == 3 else (1, int(shp[0]), int(shp[1]))
            nb = C.c_size_t()
            call("gsb_weight_images_bytes", slots, K, N, C.byref(nb))
            buf = torch.empty(int(nb.value), dtype=torch.uint8, device=self.device)
            call("gsb_weight_images_register", self._pp(name), slots, K, N, _ptr(buf), buf.numel(), _stream())
            self._wimg_bufs.append(buf)
        self._wimg_ptrs = (C.c_void_p * len(self._wimg_names))(*[self._pp(n).value for n in self._wimg_names])

    def _register_weight_images_adam(self):
        """Weight images kept current by Adam itself (gsb_adam_step_split writes the hi / lo split
        of every updated parameter into twins of the flat buffer): the layer weights' slices of
        the twins are registered as their images; no per-step refresh launch.  Computed once
        here; _params_changed() recomputes them after any write to `flat` outside Adam."""
        names = [f"W{l}" for l in range(self.L)]
        names = [n for n in names if len(self.shapes[n]) == 3 and int(self.shapes[n][2]) % 4 == 0]
        if not names:
            return
        self.flat_hi = torch.zeros_like(self.flat)
        self.flat_lo = torch.zeros_like(self.flat)
        for name in names:
            slots, K, N = (int(x) for x in self.shapes[name])
            k = self.names.index(name)
            off = int(self.offsets[k]) * 4
            call("gsb_weight_images_register_split", self._pp(name), slots, K, N,
                 C.c_void_p(self.flat_hi.data_ptr() + off), C.c_void_p(self.flat_lo.data_ptr() + off))
        self._wimg_adam = True
        # the NC decoder weight: its class-count rows are not 16-B aligned, so its image lives in
        # its own padded buffer, written by the same Adam pass (gsb_adam_step_split's segment)
        self._adam_pad = (0, 0, 0, 0, None, None)
        if "Wc" in self.names:
            K, N = (int(x) for x in self.shapes["Wc"])
            nb = C.c_size_t()
            call("gsb_weight_images_bytes", 1, K, N, C.byref(nb))
            buf = torch.zeros(int(nb.value), dtype=torch.uint8, device=self.device)
            call("gsb_weight_images_register", self._pp("Wc"), 1, K, N, _ptr(buf), buf.numel(), _stream())
            ldn = (N + 3) // 4 * 4
            self._wimg_pad_buf = buf
            self._adam_pad = (int(self.offsets[self.names.index("Wc")]), K, N, ldn, C.c_void_p(buf.data_ptr()),
                              C.c_void_p(buf.data_ptr() + K * ldn * 4))
            names = names + ["Wc"]
        self._wimg_names = names
        self._wimg_ptrs = (C.c_void_p * len(names))(*[self._pp(n).value for n in names])
        self._params_changed()

    def _params_changed(self, s=None):
        """Recompute the weight images after `flat` was written outside Adam (torch in-place
        writes to `flat` or its pview()s are detected by the tensor's version counter)."""
        if self._wimg_names:
            st = s if isinstance(s, C.c_void_p) else _stream(s)
            call("gsb_weight_images_refresh", self._wimg_ptrs, len(self._wimg_names), st)
            self._img_version = self.flat._version

    def _refresh_weight_images(self, s):
        """Start of a compute phase: images refreshed when stale (with Adam's split: only after
        writes to `flat` outside Adam)."""
        self._sync_images(s)

    def _sync_images(self, s):
        """Weight images stale only after writes to `flat` outside Adam (or without Adam's split)."""
        if not self._wimg_names:
            return
        if not getattr(self, "_wimg_adam", False):
            call("gsb_weight_images_refresh", self._wimg_ptrs, len(self._wimg_names), s)
        elif self.flat._version != getattr(self, "_img_version", -1):
            self._params_changed(s)

    def __del__(self):
        try:
            for name in getattr(self, "_wimg_names", []):
                lib().gsb_weight_images_unregister(self._pp(name))
        except Exception:
            pass

    # parameter views -------------------------------------------------------------------
    def pview(self, name: str, which: str = "p") -> torch.Tensor:
        buf = {"p": self.flat, "g": self.grad, "m": self.m, "v": self.v}[which]
        k = self.names.index(name)
        return buf[self.offsets[k]:self.offsets[k + 1]].view(self.shapes[name])

    def _pp(self, name: str, which: str = "p"):
        k = self.names.index(name)
        buf = {"p": self.flat, "g": self.grad}[which]
        return C.c_void_p(buf.data_ptr() + int(self.offsets[k]) * 4)

    # pieces ------------------------------------------------------------------------------
    def _gather_inputs(self, s):
        """Explicit input-row gather into x0 (unfused mode; with peer shards registered this is
        the unique-row NVLink fetch).  Part of the sample phase: it depends only on the blocks.
        With early_agg the input layer's aggregation (feature gather + per-relation means,
        parameter-free) runs here too, into this buffer's acat0."""
        if not self.fuse_gather and self.exchange is None and not self.enc_types:
            sm = self.sampler
            call("gsb_gather_block_inputs", sm.h, _ptr(sm.arena), _ptr(self.x0), s)
        if self.exchange is not None and not self.enc_types:
            # partitioned features, NCCL all-to-all fetch (C4/C5) into this buffer's x0 / xperm:
            # host-synced sizes, so part of the (eager) sample phase; the compute phase reads
            # the rows through the bucketing permutation
            gids, n = self.sampler.input_gids()
            self.exchange.gather(gids, n, rows_out=self.x0, perm_out=self.xperm)
        if self._early():
            sm = self.sampler
            h = None if self.fuse_gather else self.x0
            hdt = DTYPE_CODE[h.dtype] if h is not None else 0
            call("gsb_rgcn_layer_agg", sm.h, _ptr(sm.arena), 0, _ptr(h), hdt, None, self.d_in[0], _ptr(self.acat0), s)

    def _early(self) -> bool:
        return self.early_agg and not self.enc_types and self.exchange is None

    def _encode(self, s):
        """gather -> RGCN layers, input layer first (Fig. 8).  With fuse_gather
        (default) layer 0 reads the feature rows by gid inside its aggregation kernel;
        otherwise x0 was filled by _gather_inputs in the sample phase."""
        sm = self.sampler
        rowmap = None
        if self.enc_types:              # a6: projected / frozen input rows by gid -> H0 (fp32)
            call("gsb_encoder_fwd", sm.h, _ptr(sm.arena), self._win, self.d_in[0], _ptr(self.H0), _ptr(self.enc_ws),
                 self.enc_ws.numel(), s)
            for t, (E, _) in self.emb.items():     # f1: learnable tables replace the frozen rows
                if isinstance(E, _PeerTable):
                    E.pe.fwd(sm, t, self.H0, s)
                else:
                    call("gsb_sparse_emb_fwd", sm.h, _ptr(sm.arena), t, _ptr(E), self.d_in[0], _ptr(self.H0), s)
            h = self.H0
        elif self.exchange is not None:   # partitioned features fetched in the sample phase (C4/C5)
            h, rowmap = self.x0, self.xperm    # layer 0 reads rows through the bucketing permutation
        elif self.fuse_gather:
            h = None
        else:
            h = self.x0
        self.acat[0] = self.acat0
        for l in range(self.L):
            if l == 0 and self._early():   # acat0 was filled in the sample phase
                call("gsb_rgcn_layer_gemm", sm.h, _ptr(sm.arena), 0, _ptr(self.acat0), self.d_in[0],
                     self._pp("W0"), self._pp("b0"), self.hidden, int(self.L > 1), _ptr(self.hout[0]), s)
            else:
                hdt = DTYPE_CODE[h.dtype] if h is not None else 0
                call("gsb_rgcn_layer_fwd_ex", sm.h, _ptr(sm.arena), l, _ptr(h), hdt, _ptr(rowmap if l == 0 else None),
                     self.d_in[l], self._pp(f"W{l}"), self._pp(f"b{l}"), self.hidden, int(l < self.L - 1),
                     _ptr(self.hout[l]), _ptr(self.acat[l]), s)
            h = self.hout[l]
        return h

    def _step_body(self, stream=None, step: int = 0, step_dev=None, seeds=None):
        """One step without the optimizer: sample phase, then compute phase."""
        self._sample_phase(stream, step, step_dev, seeds)
        self._compute_phase(stream, seeds)

    def _backward_layers(self, s):
        sm = self.sampler
        for l in reversed(range(self.L)):
            dh_src = (self.dH0 if self.enc_types else None) if l == 0 else self.dh[l - 1]
            call("gsb_rgcn_layer_bwd", sm.h, _ptr(sm.arena), l, _ptr(self.hout[l]), _ptr(self.dh[l]),
                 self._pp(f"W{l}"), _ptr(self.acat[l]), self.d_in[l], self.hidden, int(l < self.L - 1),
                 self._pp(f"W{l}", "g"), self._pp(f"b{l}", "g"), _ptr(dh_src),
                 _ptr(self.dacat) if dh_src is not None else None, s)
        if self.enc_types:   # a6 backward: dWin_t = X_t^T dH0 (frozen tables get no gradient)
            call("gsb_encoder_bwd", sm.h, _ptr(sm.arena), self._win, _ptr(self.dH0), self.d_in[0], self._dwin,
                 _ptr(self.enc_ws), self.enc_ws.numel(), s)

    def set_embedding(self, ntype: int, E: torch.Tensor, lr: float = 0.01, eps: float = 1e-10, peers=None):
        """Make ntype's input rows a learnable table (§8(f) f1): E fp32 [N_t][d_in0] (copied),
        trained by sparse Adagrad on the rows each mini-batch touches (gsb_sparse_adagrad).
        Needs the input-encoder path (H0) and a non-projected ntype.  peers: a
        dist.PeerEmbedding holding the table partitioned over the ranks (R-sparsedist);
        otherwise this GPU holds all of it."""
        if not self.enc_types or ntype in self.enc_types:
            raise _lib.GsbError("learnable embeddings need the encoder path and a non-projected ntype")
        if E.shape != (int(self.store.counts[ntype]), self.d_in[0]):
            raise _lib.GsbError(f"embedding table shape {tuple(E.shape)}")
        if peers is not None:
            self.emb[ntype] = (_PeerTable(peers), None)
        else:
            E = E.to(self.device, torch.float32).contiguous().clone()
            self.emb[ntype] = (E, torch.zeros_like(E))
        self.emb_lr, self.emb_eps = lr, eps

    def _peer_push(self, stream=None):
        """N > 1: push the partitioned tables' gradients before the dense all-reduce, which
        then doubles as the barrier between every rank's push and the owners' apply."""
        for t, (E, _) in self.emb.items():
            if isinstance(E, _PeerTable):
                E.pe.push(self.sampler, t, self.dH0, _stream(stream))
                self._pushed = True

    def _sparse_update(self, stream=None):
        sm = self.sampler
        pushed = getattr(self, "_pushed", False)
        self._pushed = False
        for t, (E, st) in self.emb.items():
            if isinstance(E, _PeerTable):
                E.pe.update(sm, t, self.dH0, self.emb_lr, self.emb_eps, _stream(stream), pushed=pushed)
                continue
            call("gsb_sparse_adagrad", sm.h, _ptr(sm.arena), t, _ptr(E), _ptr(st), _ptr(self.dH0), self.d_in[0],
                 self.emb_lr, self.emb_eps, _stream(stream))

    def optimizer_step(self, stream=None, t_dev: bool = False):
        self._sparse_update(stream)
        t_ptr = C.c_void_p(self.counters.data_ptr() + 4) if t_dev else None
        if not t_dev:
            self.t += 1
        t = 1 if t_dev else self.t
        if self.flat_hi is not None:      # Adam also refreshes the GEMMs' weight images
            call("gsb_adam_step_split", _ptr(self.flat), _ptr(self.grad), _ptr(self.m), _ptr(self.v), self.n_params,
                 self.lr, 0.9, 0.999, 1e-8, t, t_ptr, _ptr(self.flat_hi), _ptr(self.flat_lo), *self._adam_pad,
                 _stream(stream))
        else:
            call("gsb_adam_step", _ptr(self.flat), _ptr(self.grad), _ptr(self.m), _ptr(self.v), self.n_params,
                 self.lr, 0.9, 0.999, 1e-8, t, t_ptr, _stream(stream))

    # CUDA graph of one whole step ----------------------------------------------------------
    def capture(self, step0: int, ws: int = 1, allreduce=None):
        """Capture one step in a CUDA graph reading its inputs from the fixed input buffers and
        the RNG step / Adam t from device counters, which the graph advances (step += ws,
        t += 1).  Single GPU: sample..Adam in the graph.  With `allreduce` (N>1) the graph
        ends at the gradients; replay() then runs the NCCL all-reduce and Adam eagerly (NCCL
        is kept out of graph capture).  Subsequent steps: load inputs, then replay()."""
        self.graph_allreduce = allreduce
        self.counters[0] = step0
        self.counters[1] = self.t
        self.graph_ws = ws
        self._sync_images(_stream())   # images current before capture (none captured)
        torch.cuda.synchronize()
        launches0 = lib().gsb_launch_count()
        g = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            with torch.cuda.graph(g, stream=side):
                s = _stream()
                call("gsb_counter_add", C.c_void_p(self.counters.data_ptr() + 4), 1, s)
                self._step_body(stream=None, step=0, step_dev=self.counters[0:1])
                if allreduce is None:
                    self.optimizer_step(t_dev=True)
                call("gsb_counter_add", C.c_void_p(self.counters.data_ptr()), ws, s)
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        self.graph_launches = lib().gsb_launch_count() - launches0
        self.graph = g
        return g

    def replay(self):
        self._sync_images(_stream())   # only if flat was written since (version check)
        self.graph.replay()
        if self.graph_allreduce is not None:
            self._peer_push()
            self.graph_allreduce(self.grad)
            self.optimizer_step(t_dev=True)
        self.t += 1

    # double-buffered pipeline: sample batch i+1 while batch i computes ---------------------
    _BUFFERED = ("sampler", "x0", "acat0", "xperm")   # per-batch state; subclasses add their input buffers

    def enable_prefetch(self):
        """Allocate a second copy of every per-batch buffer (sampler handle + arena, input
        rows, the task's input tensors) so the sample phase of batch i+1 -- sampling,
        relabel and, in unique-gather mode, the input-row fetch; none of it reads the
        parameters -- runs on a side stream while batch i computes."""
        if self._bufs is not None:
            return
        cur = {k: getattr(self, k) for k in self._BUFFERED}
        nxt = {k: (v.twin() if isinstance(v, MiniBatchSampler) else torch.zeros_like(v)) for k, v in cur.items()}
        self._bufs = [cur, nxt]
        # Stream priorities (A/B knob, profiles/round1e_stream_priority.md): GSB_PRIO=1 replays the
        # compute phase on a high-priority stream, 2 gives the sample side stream the high
        # priority, 0 (default) keeps both at the default priority.
        prio = os.environ.get("GSB_PRIO", "0")
        self.side = torch.cuda.Stream(device=self.device, priority=-1 if prio == "2" else 0)
        self.hi = torch.cuda.Stream(device=self.device, priority=-1) if prio == "1" else None
        self.ev_s = [torch.cuda.Event(), torch.cuda.Event()]
        self.ev_c = torch.cuda.Event()

    def _use(self, b: int):
        for k, v in self._bufs[b].items():
            setattr(self, k, v)
        self.acat[0] = self.acat0

    def _sample_ops(self):
        """Sample phase of the batch in the active buffer, RNG step word read from (and then
        advanced on) the device counter."""
        self._sample_phase(None, 0, self.counters[0:1])
        call("gsb_counter_add", C.c_void_p(self.counters.data_ptr()), self.pipe_ws, _stream())

    def _compute_ops(self):
        call("gsb_counter_add", C.c_void_p(self.counters.data_ptr() + 4), 1, _stream())
        self._compute_phase(None)
        if self.pipe_allreduce is None:
            self.optimizer_step(t_dev=True)

    def pipeline_start(self, inputs, step: int, ws: int = 1, allreduce=None, use_graph: bool = True):
        """Start a pipelined run: capture (once) per-buffer CUDA graphs of the sample phase
        and of the compute phase (+ Adam unless `allreduce`, which then runs eagerly after
        each compute graph, NCCL being kept out of capture), then load `inputs` (the first
        batch) into buffer 0 and sample it with RNG step word `step`.  Each pipeline_step()
        computes the pending batch and samples the next one (step word + ws)."""
        if self.exchange is not None:   # host-synced all-to-all sizes: eager sample phase
            self.sample_graph = False
        self.enable_prefetch()
        self.pipe_ws, self.pipe_allreduce = ws, allreduce
        self._sync_images(_stream())   # images current before capture (none captured)
        sample_graph = getattr(self, "sample_graph", True)   # False: NCCL frontier exchange (host-synced)
        if use_graph and self.pipe_graphs is None:
            torch.cuda.synchronize()
            launches0 = lib().gsb_launch_count()
            cap = torch.cuda.Stream(device=self.device)
            graphs = {"sample": [], "compute": []}
            kinds = (("sample", self._sample_ops), ("compute", self._compute_ops)) if sample_graph else \
                (("compute", self._compute_ops),)
            for kind, fn in kinds:
                for b in (0, 1):
                    g = torch.cuda.CUDAGraph()
                    cap.wait_stream(torch.cuda.current_stream())
                    with torch.cuda.stream(cap):
                        with torch.cuda.graph(g, stream=cap):
                            self._use(b)
                            fn()
                    torch.cuda.current_stream().wait_stream(cap)
                    graphs[kind].append(g)
            torch.cuda.synchronize()
            # kernels per step = one sample graph + one compute graph
            self.graph_launches = (lib().gsb_launch_count() - launches0) // 2
            self.pipe_graphs = graphs if sample_graph else dict(graphs, sample=None)
        elif not use_graph:
            self.pipe_graphs = None
        self.pipe_k = 0
        self.counters[0] = step + ws
        self.counters[1] = self.t
        self._use(0)
        self._load_inputs(self._bufs[0], *inputs)
        self._sample_phase(None, step, None)
        self.ev_s[0].record()
        self.ev_c.record()

    def pipeline_step(self, *next_inputs):
        """Compute the pending batch (loss, grads, Adam) on the current stream while the side
        stream loads `next_inputs` into the other buffer and samples them.  Afterwards
        self.loss is the computed batch's loss (read it on the current stream)."""
        b = self.pipe_k & 1
        nb = b ^ 1
        main = torch.cuda.current_stream()
        self._sync_images(_stream())   # only if flat was written since (version check)

        def sample_next():
            self.side.wait_event(self.ev_c)          # buffer nb is free once batch k-1 computed
            with torch.cuda.stream(self.side):
                self._load_inputs(self._bufs[nb], *next_inputs)
                if self.pipe_graphs is not None and self.pipe_graphs["sample"] is not None:
                    self.pipe_graphs["sample"][nb].replay()
                else:
                    self._use(nb)
                    self._sample_ops()
                self.ev_s[nb].record(self.side)

        cs = main if self.hi is None else self.hi

        def compute():
            if cs is not main:
                cs.wait_stream(main)
            cs.wait_event(self.ev_s[b])
            self._use(b)
            with torch.cuda.stream(cs):
                if self.pipe_graphs is not None:
                    self.pipe_graphs["compute"][b].replay()
                else:
                    self._compute_ops()
            if cs is not main:
                main.wait_stream(cs)

        if getattr(self, "sample_graph", True):
            sample_next()
            compute()
        else:
            # host-synced sampling (NCCL exchange): enqueue the compute graph first, so the host
            # waits inside the exchange while batch k computes on the device
            compute()
            sample_next()
            self._use(b)
        if self.pipe_allreduce is not None:
            # the sparse table update (N > 1, after the all-reduce) still reads buffer b's block:
            # the side stream may overwrite b (batch k+2) only after it
            if not self.emb:
                self.ev_c.record(main)
            self._peer_push()
            self.pipe_allreduce(self.grad)
            self.optimizer_step(t_dev=True)
            if self.emb:
                self.ev_c.record(main)
        else:
            self.ev_c.record(main)
        self.t += 1
        self.pipe_k += 1

    def pipeline_sync(self):
        """Join the side stream into the current stream (end of a pipelined run)."""
        if self._bufs is not None:
            torch.cuda.current_stream().wait_stream(self.side)


class RGCNTrainer(_TrainerBase):
    """Node classification (§8(a) a1-a8, a11, a12): RGCN encoder + softmax-CE decoder.

    params (synth.init_params layout): W{l} (R+1, d_in, d_out), b{l}, Wc (hidden, C), bc.
    """

    def __init__(self, store: GraphStore, fanouts: Sequence[int], batch: int, hidden: int, num_classes: int,
                 params: Dict[str, np.ndarray], param_order: Sequence[str], labels: torch.Tensor,
                 label_gid_base: int, lr: float = 1e-3, rng_seed: int = 1):
        super().__init__(store, fanouts, batch, hidden, params, param_order, lr, rng_seed)
        dev = store.device
        self.batch = batch
        self.C = num_classes
        self.labels = labels.to(dev, dtype=torch.int32).contiguous()
        self.label_base = int(label_gid_base)
        self.logits = torch.empty((batch, (max(num_classes, 1) + 3) // 4 * 4), dtype=torch.float32, device=dev)
        self.row_loss = torch.zeros(batch + 640, dtype=torch.float32, device=dev)   # + fused-mean scratch
        self.seeds_dev = torch.empty(batch, dtype=torch.int64, device=dev)
        # the decoder weight gradient (gsb_nc_loss_dw) on a stream of its own, joined after the
        # layers' backward instead of inside gsb_nc_loss (GSB_DWC_SIDE=0: joined inside)
        self.dwc_stream = (torch.cuda.Stream(device=dev) if os.environ.get("GSB_DWC_SIDE", "1") != "0"
                           else None)
        self.dwc_ws = (torch.empty(hidden * self.logits.shape[1], dtype=torch.float32, device=dev)
                       if os.environ.get("GSB_DWC_PAD", "1") != "0" else None)

    _BUFFERED = ("sampler", "x0", "acat0", "xperm", "seeds_dev")

    def _load_inputs(self, d, seeds: torch.Tensor):
        d["seeds_dev"][:seeds.numel()].copy_(seeds, non_blocking=True)

    def _sample_phase(self, stream=None, step: int = 0, step_dev=None, seeds=None):
        seeds = self.seeds_dev if seeds is None else seeds
        self.sampler.sample(seeds, self.rng_seed, step, stream=stream, step_dev=step_dev)
        self._gather_inputs(_stream(stream))

    def _compute_phase(self, stream=None, seeds=None):
        s = _stream(stream)
        self._refresh_weight_images(s)
        seeds = self.seeds_dev if seeds is None else seeds
        n = seeds.numel()
        h = self._encode(s)
        top = self.L - 1
        side = self.dwc_stream
        call("gsb_nc_loss", _ptr(h), n, self.hidden, self._pp("Wc"), self._pp("bc"), self.C, _ptr(self.labels),
             _ptr(seeds), self.label_base, _ptr(self.logits), _ptr(self.row_loss), _ptr(self.loss),
             _ptr(self.dh[top]), None if side else self._pp("Wc", "g"), None if side else self._pp("bc", "g"), s)
        if side is not None:
            main = stream if stream is not None else torch.cuda.current_stream()
            side.wait_stream(main)
            call("gsb_nc_loss_dw", _ptr(h), n, self.hidden, _ptr(self.logits), self.C, self._pp("Wc", "g"),
                 self._pp("bc", "g"), _ptr(self.dwc_ws), _stream(side))
        self._backward_layers(s)
        if side is not None:
            main.wait_stream(side)

    def forward_backward(self, seeds: torch.Tensor, step: int, stream=None):
        """Sample -> gather -> layers (input layer first) -> NC loss -> backward."""
        self._step_body(stream, step, None, seeds)

    def train_step(self, seeds: torch.Tensor, step: int, stream=None):
        self.forward_backward(seeds, step, stream)
        self.optimizer_step(stream)

    def load_inputs(self, seeds: torch.Tensor):
        self.seeds_dev[:seeds.numel()].copy_(seeds, non_blocking=True)

    def train_step_host(self, seeds_host: torch.Tensor, step: int, loss_host: torch.Tensor,
                        eager: bool = False) -> float:
        """Public end-to-end call: seeds from (pinned) host memory, loss back to the host.
        Uses the captured CUDA graph when one exists (the step word then comes from the
        device counter, advanced by each replay)."""
        n = seeds_host.numel()
        dst = self.seeds_dev[:n]
        dst.copy_(seeds_host, non_blocking=True)
        if self.graph is not None and n == self.batch and not eager:
            self.replay()
        else:
            self.train_step(dst, step)
        loss_host.copy_(self.loss, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return float(loss_host[0])


class LPTrainer(_TrainerBase):
    """Link prediction (§8(a) a3', a9, a10; §8(f) f2): negatives, target-edge exclusion,
    RGCN encoder, DistMult / dot-product score, contrastive / CE / weighted CE loss.
    params: W{l}, b{l}, rel (DistMult).

    neg_sampler (App. A.2.1): "joint" (K nodes per group of K positives),
    "uniform" (K per positive), "local_joint" (joint over local_range = (first local id,
    count) of the dst type: this rank's partition), "in_batch" (the other positives'
    destinations, K = B - 1, nothing drawn)."""

    def __init__(self, store: GraphStore, fanouts: Sequence[int], batch: int, hidden: int, num_neg: int,
                 lp_etype: int, lp_rev_etype: int, params: Dict[str, np.ndarray], param_order: Sequence[str],
                 lr: float = 1e-3, rng_seed: int = 1, loss_kind: int = 0, neg_sampler: str = "joint",
                 score: str = "distmult", local_range=None):
        B = batch
        if neg_sampler not in ("joint", "uniform", "local_joint", "in_batch"):
            raise _lib.GsbError(f"unknown negative sampler {neg_sampler!r}")
        if score not in ("distmult", "dot"):
            raise _lib.GsbError(f"unknown score {score!r}")
        K = B - 1 if neg_sampler == "in_batch" else num_neg
        self.neg_sampler, self.score = neg_sampler, score
        self.neg_mode = 1 if neg_sampler == "in_batch" else 0
        self.group = 1 if neg_sampler == "uniform" else K
        if neg_sampler == "in_batch":
            self.n_neg = 0
        elif neg_sampler == "uniform":
            self.n_neg = B * K
        else:
            self.n_neg = ((B + K - 1) // K) * K
        self.G = (B + K - 1) // K
        max_seeds = 2 * B + self.n_neg
        super().__init__(store, fanouts, max_seeds, hidden, params, param_order, lr, rng_seed, max_excl=B)
        dev = store.device
        self.B, self.K = B, K
        self.lp_etype, self.lp_rev = lp_etype, lp_rev_etype
        self.loss_kind = loss_kind
        dst_t = int(store.etype_dst[lp_etype])
        self.neg_base = int(store.node_off[dst_t])
        self.neg_n = int(store.counts[dst_t])
        if neg_sampler == "local_joint" and local_range is not None:
            self.neg_base += int(local_range[0])
            self.neg_n = int(local_range[1])
        self.pos_u = torch.empty(B, dtype=torch.int64, device=dev)
        self.pos_v = torch.empty(B, dtype=torch.int64, device=dev)
        self.neg = torch.empty(max(self.n_neg, 1), dtype=torch.int64, device=dev)
        self.seeds = torch.empty(max_seeds, dtype=torch.int64, device=dev)
        self.n_seeds = torch.zeros(1, dtype=torch.int64, device=dev)
        self.iu = torch.empty(B, dtype=torch.int32, device=dev)
        self.iv = torch.empty(B, dtype=torch.int32, device=dev)
        self.ineg = torch.empty(max(self.n_neg, 1), dtype=torch.int32, device=dev)
        self.pos_w = torch.ones(B, dtype=torch.float32, device=dev)    # Eq. 5 weights (loss_kind 2)
        # the input aggregation stays in the compute phase (GSB_LP_EARLY=1 moves it to the sample
        # phase as for NC: the phases swap lengths but the overlapped step gets slower, 1.2753 ->
        # 1.3053 ms on amazon_lp, gpurun_out/lp1: the two streams share the SMs either way)
        self.early_agg = os.environ.get("GSB_LP_EARLY", "0") == "1"
        wb = C.c_size_t()
        call("gsb_lp_seeds_bytes", B, self.n_neg, C.byref(wb))
        self.seeds_ws = torch.empty(int(wb.value), dtype=torch.uint8, device=dev)
        self.scores = torch.empty((B, K + 1), dtype=torch.float32, device=dev)
        self.row_loss = torch.empty(B, dtype=torch.float32, device=dev)
        call("gsb_lp_score_ws_bytes", B, hidden, self.neg_mode, C.byref(wb))
        self.score_ws = torch.empty(max(int(wb.value), 1), dtype=torch.uint8, device=dev)
        self.group_base = 0
        self.pos_base = 0

    _BUFFERED = ("sampler", "x0", "acat0", "xperm", "pos_u", "pos_v", "neg", "seeds", "n_seeds", "iu", "iv", "ineg",
                 "seeds_ws")

    def _load_inputs(self, d, u: torch.Tensor, v: torch.Tensor):
        d["pos_u"].copy_(u, non_blocking=True)
        d["pos_v"].copy_(v, non_blocking=True)

    def _sample_phase(self, stream=None, step: int = 0, step_dev=None, seeds=None):
        """Joint negatives -> LP seed set -> exclusion-aware sampling (-> input rows)."""
        s = _stream(stream)
        sd = None if step_dev is None else C.c_void_p(step_dev.data_ptr())
        if self.neg_sampler in ("joint", "local_joint"):
            call("gsb_joint_negatives", self.B, self.K, self.neg_n, self.neg_base, self.rng_seed, step, sd,
                 self.group_base, _ptr(self.neg), s)
        elif self.neg_sampler == "uniform":
            call("gsb_uniform_negatives", self.B, self.K, self.neg_n, self.neg_base, self.rng_seed, step, sd,
                 self.pos_base, _ptr(self.neg), s)
        has_neg = self.n_neg > 0
        call("gsb_lp_seeds", _ptr(self.pos_u), _ptr(self.pos_v), self.B, _ptr(self.neg) if has_neg else None,
             self.n_neg, _ptr(self.seeds), _ptr(self.n_seeds), _ptr(self.iu), _ptr(self.iv),
             _ptr(self.ineg) if has_neg else None, _ptr(self.seeds_ws), self.seeds_ws.numel(), s)
        self.sampler.sample(self.seeds, self.rng_seed, step, self.pos_u, self.pos_v, self.lp_etype, self.lp_rev, stream,
                            n_seeds_dev=self.n_seeds, step_dev=step_dev, n_seeds=self.seeds.numel())
        self._gather_inputs(s)

    def _compute_phase(self, stream=None, seeds=None):
        s = _stream(stream)
        self._refresh_weight_images(s)
        h = self._encode(s)
        top = self.L - 1
        dm = self.score == "distmult"
        call("gsb_lp_score_ex", _ptr(h), self.hout[top].shape[0], self.hidden, _ptr(self.iu), _ptr(self.iv),
             _ptr(self.ineg) if self.n_neg > 0 else None, self.B, self.K, self.group, self.neg_mode,
             self._pp("rel") if dm else None, self.loss_kind, _ptr(self.pos_w), _ptr(self.scores),
             _ptr(self.row_loss), _ptr(self.loss), _ptr(self.dh[top]), self._pp("rel", "g") if dm else None,
             _ptr(self.score_ws), self.score_ws.numel(), s)
        self._backward_layers(s)

    def mrr(self, stream=None) -> torch.Tensor:
        """MRR (R-mrr) of the last step's scores (each positive ranked among its K
        negatives; gsb_lp_mrr).  Returns a device fp32 scalar; per-positive reciprocal
        ranks in self.rr."""
        if not hasattr(self, "rr"):
            self.rr = torch.empty(self.B, dtype=torch.float32, device=self.scores.device)
            self.mrr_dev = torch.empty(1, dtype=torch.float32, device=self.scores.device)
        call("gsb_lp_mrr", _ptr(self.scores), self.scores.shape[1], self.B, self.K, _ptr(self.rr),
             _ptr(self.mrr_dev), _stream(stream))
        return self.mrr_dev

    def load_inputs(self, u: torch.Tensor, v: torch.Tensor):
        self.pos_u.copy_(u, non_blocking=True)
        self.pos_v.copy_(v, non_blocking=True)

    def forward_backward(self, u: torch.Tensor, v: torch.Tensor, step: int, stream=None):
        self.load_inputs(u, v)
        self._step_body(stream, step)

    def train_step(self, u: torch.Tensor, v: torch.Tensor, step: int, stream=None):
        self.forward_backward(u, v, step, stream)
        self.optimizer_step(stream)


class FullGraphInference:
    """Full-graph layer-wise inference (P:L393 --inference, P:L403
    --save-embed-path): h_l of every node over its whole in-neighbourhood, layer by layer, in
    chunks of consecutive gids (fanout ALL, one-layer blocks).  Every arithmetic step runs in
    libgsb (gsb_sample, gsb_rgcn_layer_fwd_ex, gsb_blocks_input_rowmap, gsb_nc_predict);
    torch holds the all-node tables.  params: W{l}, b{l} (and Wc, bc for predict)."""

    def __init__(self, store: GraphStore, params: Dict[str, np.ndarray], num_layers: int, hidden: int,
                 chunk: int = 1 << 16):
        if any(k.startswith("Win") for k in params):
            raise _lib.GsbError("full-graph inference with an input encoder is not supported yet")
        self.store, self.L, self.hidden = store, num_layers, hidden
        self.chunk = int(min(chunk, int(store.node_off[-1])))
        dev = store.device
        self.p = {k: torch.from_numpy(np.ascontiguousarray(v, np.float32)).to(dev) for k, v in params.items()}
        self.sampler = MiniBatchSampler(store, [-1], self.chunk)
        self.N = int(store.node_off[-1])
        self.d_in = [int(params["W0"].shape[1])] + [hidden] * (num_layers - 1)
        nin = self.sampler.input_rows()
        self.rowmap = torch.empty(nin, dtype=torch.int32, device=dev)
        self.acat = torch.empty(max(self.sampler.acat_floats(0, d) for d in self.d_in), dtype=torch.float32,
                                device=dev)
        self.H: List[torch.Tensor] = []

    def run(self, stream=None) -> torch.Tensor:
        """All layers; returns the last layer's table [N_total][hidden] (fp32, device)."""
        s = _stream(stream)
        sm = self.sampler
        dev = self.store.device
        self.H = []
        h_prev = None
        for l in range(self.L):
            H = torch.empty((self.N, self.hidden), dtype=torch.float32, device=dev)
            for a in range(0, self.N, self.chunk):
                b = min(a + self.chunk, self.N)
                seeds = torch.arange(a, b, dtype=torch.int64, device=dev)
                sm.sample(seeds, 0, 0, stream=stream)
                rm = None
                if h_prev is not None:
                    call("gsb_blocks_input_rowmap", sm.h, _ptr(sm.arena), 0, _ptr(self.rowmap), s)
                    rm = self.rowmap
                call("gsb_rgcn_layer_fwd_ex", sm.h, _ptr(sm.arena), 0, _ptr(h_prev),
                     0 if h_prev is None else DTYPE_CODE[torch.float32], _ptr(rm), self.d_in[l],
                     _ptr(self.p[f"W{l}"]), _ptr(self.p[f"b{l}"]), self.hidden, int(l < self.L - 1),
                     _ptr(H[a:b]), _ptr(self.acat), s)
            self.H.append(H)
            h_prev = H
        return self.H[-1]

    def predict(self, gids: torch.Tensor, labels: torch.Tensor, label_gid_base: int, num_classes: int,
                stream=None):
        """NC decoder over the given nodes' final embeddings: (pred int32 [n], #correct)."""
        h = self.H[-1].index_select(0, gids)     # row selection (plumbing)
        n = int(gids.numel())
        C_pad = (num_classes + 3) // 4 * 4
        logits = torch.empty((max(n, 1), C_pad), dtype=torch.float32, device=h.device)
        pred = torch.empty(max(n, 1), dtype=torch.int32, device=h.device)
        correct = torch.zeros(1, dtype=torch.int64, device=h.device)
        lab = labels.to(h.device, torch.int32).contiguous()
        call("gsb_nc_predict", _ptr(h), n, self.hidden, _ptr(self.p["Wc"]), _ptr(self.p["bc"]), num_classes,
             _ptr(lab), _ptr(gids), label_gid_base, _ptr(logits), _ptr(pred), _ptr(correct), _stream(stream))
        return pred[:n], int(correct.item())

    def save(self, path: str):
        """Embedding export (P:L403 --save-embed-path): the last layer's table as .npy."""
        np.save(path, self.H[-1].cpu().numpy())
