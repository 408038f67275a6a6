"""Thin Python driver over libgsb: device memory (torch tensors), streams, and the order of
C-ABI calls that make one RGCN mini-batch train step (Fig. 4; Fig. 8
P:L480-489).  Every arithmetic step runs in libgsb's CUDA kernels; this module only
allocates buffers and passes pointers.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import call, lib


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream(stream: Optional[torch.cuda.Stream] = None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _require_cuda():
    if not torch.cuda.is_available():
        raise _lib.GsbError("libgsb needs a CUDA device (there is no CPU fallback)")


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

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().gsb_graph_destroy(self.h)
        except Exception:
            pass

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

    def set_features(self, t: int, feat: torch.Tensor):
        f = feat.to(self.device, dtype=torch.float32).contiguous()
        call("gsb_graph_set_features", self.h, t, _ptr(f), f.shape[1])
        self.feats[t] = f
        self.feat_dim = f.shape[1]

    def gather(self, gids: torch.Tensor) -> torch.Tensor:
        """gsb_gather: out[i] = F_{t(i)}[gid_i - off_t]."""
        g = gids.to(self.device, dtype=torch.int64).contiguous()
        out = torch.empty((g.numel(), self.feat_dim), dtype=torch.float32, device=self.device)
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

    def __del__(self):
        try:
            if getattr(self, "h", None):
                lib().gsb_blocks_destroy(self.h)
        except Exception:
            pass

    def sample(self, seeds: torch.Tensor, rng_seed: int, step: int, excl_u: Optional[torch.Tensor] = None,
               excl_v: Optional[torch.Tensor] = None, excl_etype: int = -1, excl_rev_etype: int = -1,
               stream=None):
        n_ex = 0 if excl_u is None else excl_u.numel()
        call("gsb_sample", self.h, _ptr(seeds), seeds.numel(), rng_seed, step, _ptr(excl_u), _ptr(excl_v), n_ex,
             excl_etype, excl_rev_etype, _ptr(self.arena), self.arena.numel(), _stream(stream))

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


class RGCNTrainer:
    """One RGCN mini-batch train step through libgsb (§8(a) a1-a12, NC task).

    params: dict name -> float32 numpy (synth.init_params layout: W{l} (R+1, d_in, d_out),
    b{l}, Wc, bc).  All parameters live in one flat fp32 device buffer (one Adam launch).
    """

    def __init__(self, store: GraphStore, fanouts: Sequence[int], batch: int, hidden: int, num_classes: int,
                 params: Dict[str, np.ndarray], param_order: Sequence[str], labels: torch.Tensor,
                 label_gid_base: int, lr: float = 1e-3, rng_seed: int = 1):
        self.store = store
        self.L = len(fanouts)
        self.batch = batch
        self.hidden = hidden
        self.C = num_classes
        self.lr = lr
        self.rng_seed = rng_seed
        self.sampler = MiniBatchSampler(store, fanouts, max_seeds=batch)
        dev = store.device
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
        self.labels = labels.to(dev, dtype=torch.int32).contiguous()
        self.label_base = int(label_gid_base)
        d0 = store.feat_dim
        self.d_in = [d0] + [hidden] * (self.L - 1)
        # activations / caches (upper-bound sized; never reallocated)
        self.x0 = torch.empty((self.sampler.input_rows(), d0), dtype=torch.float32, device=dev)
        self.hout = [torch.empty((self.sampler.dst_rows(l), hidden), dtype=torch.float32, device=dev)
                     for l in range(self.L)]
        self.acat = [torch.empty(self.sampler.acat_floats(l, self.d_in[l]), dtype=torch.float32, device=dev)
                     for l in range(self.L)]
        self.dacat = torch.empty(max(self.sampler.acat_floats(l, self.d_in[l]) for l in range(self.L)),
                                 dtype=torch.float32, device=dev)
        self.dh = [torch.empty((self.sampler.dst_rows(l), hidden), dtype=torch.float32, device=dev)
                   for l in range(self.L)]
        self.logits = torch.empty((batch, max(num_classes, 1)), dtype=torch.float32, device=dev)
        self.row_loss = torch.empty(batch, dtype=torch.float32, device=dev)
        self.loss = torch.zeros(1, dtype=torch.float32, device=dev)
        self.seeds_dev = torch.empty(batch, dtype=torch.int64, device=dev)

    # parameter views -------------------------------------------------------------------
    def pview(self, name: str, which: str = "p") -> torch.Tensor:
        buf = {"p": self.flat, "g": self.grad, "m": self.m, "v": self.v}[which]
        k = self.names.index(name)
        return buf[self.offsets[k]:self.offsets[k + 1]].view(self.shapes[name])

    def _pp(self, name: str, which: str = "p"):
        k = self.names.index(name)
        buf = {"p": self.flat, "g": self.grad}[which]
        return C.c_void_p(buf.data_ptr() + int(self.offsets[k]) * 4)

    # the step ----------------------------------------------------------------------------
    def forward_backward(self, seeds: torch.Tensor, step: int, stream=None):
        """Sample -> gather -> layers (input layer first) -> NC loss -> backward."""
        s = _stream(stream)
        n = seeds.numel()
        self.sampler.sample(seeds, self.rng_seed, step, stream=stream)
        sm = self.sampler
        call("gsb_gather_block_inputs", sm.h, _ptr(sm.arena), _ptr(self.x0), s)
        h = self.x0
        for l in range(self.L):
            call("gsb_rgcn_layer_fwd", sm.h, _ptr(sm.arena), l, _ptr(h), self.d_in[l], self._pp(f"W{l}"),
                 self._pp(f"b{l}"), self.hidden, int(l < self.L - 1), _ptr(self.hout[l]), _ptr(self.acat[l]), s)
            h = self.hout[l]
        top = self.L - 1
        call("gsb_nc_loss", _ptr(h), n, self.hidden, self._pp("Wc"), self._pp("bc"), self.C, _ptr(self.labels),
             _ptr(seeds), self.label_base, _ptr(self.logits), _ptr(self.row_loss), _ptr(self.loss),
             _ptr(self.dh[top]), self._pp("Wc", "g"), self._pp("bc", "g"), s)
        for l in reversed(range(self.L)):
            h_src = self.x0 if l == 0 else self.hout[l - 1]
            dh_src = None if l == 0 else self.dh[l - 1]
            call("gsb_rgcn_layer_bwd", sm.h, _ptr(sm.arena), l, _ptr(self.hout[l]), _ptr(self.dh[l]),
                 self._pp(f"W{l}"), _ptr(self.acat[l]), self.d_in[l], self.hidden, int(l < self.L - 1),
                 self._pp(f"W{l}", "g"), self._pp(f"b{l}", "g"), _ptr(dh_src),
                 _ptr(self.dacat) if dh_src is not None else None, s)
            del h_src

    def optimizer_step(self, stream=None):
        self.t += 1
        call("gsb_adam_step", _ptr(self.flat), _ptr(self.grad), _ptr(self.m), _ptr(self.v), self.n_params, self.lr,
             0.9, 0.999, 1e-8, self.t, _stream(stream))

    def train_step(self, seeds: torch.Tensor, step: int, stream=None):
        """One full step on device-resident seeds; returns nothing (loss stays on device)."""
        self.forward_backward(seeds, step, stream)
        self.optimizer_step(stream)

    def train_step_host(self, seeds_host: torch.Tensor, step: int, loss_host: torch.Tensor) -> float:
        """Public end-to-end call: seeds from (pinned) host memory, loss back to the host."""
        n = seeds_host.numel()
        dst = self.seeds_dev[:n]
        dst.copy_(seeds_host, non_blocking=True)
        self.train_step(dst, step)
        loss_host.copy_(self.loss, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return float(loss_host[0])
