"""Multi-GPU plumbing (one process per GPU, torch.distributed): synchronous data parallel
with mean-reduced dense gradients (§8(a) a12; S:L308-311 all_reduce_gradients) and the
per-rank batch assignment.  Collectives are NCCL on GPUs (gloo in the CPU tests); the
arithmetic of a step stays in libgsb.
"""
from __future__ import annotations

from typing import Optional

import torch


def allreduce_mean(t: torch.Tensor, group=None, world: Optional[int] = None) -> torch.Tensor:
    """In place: t <- mean over ranks of t.  NCCL: one ncclAvg all-reduce (the 1/world scale
    happens inside the collective, no extra kernel); gloo (CPU tests) has no AVG: sum, then
    scale by 1/world."""
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        dist.all_reduce(t, op=dist.ReduceOp.AVG, group=group)
        return t
    ws = world if world is not None else dist.get_world_size(group)
    dist.all_reduce(t, group=group)
    if ws > 1:
        t.mul_(1.0 / ws)
    return t


def rank_step(step: int, rank: int, world: int) -> int:
    """Global batch index of `step` on `rank`: rank r takes batches step*world + r, so the
    union over ranks of one step is `world` consecutive batches (a round-robin split of a
    global batch) and the RNG step word (keyed sampling) stays globally unique."""
    return step * world + rank


def balanced_bounds(counts, world: int):
    """Contiguous node-ID ranges per ntype (random partition: the generator scatters node
    ranks by an affine bijection).  bounds[t][w] = floor(N_t * w / world)."""
    import numpy as np
    return np.array([[(int(n) * w) // world for w in range(world + 1)] for n in counts], dtype=np.int64)


class FeatureExchange:
    """Partitioned feature store (§8(e)): this rank holds only its node-ID range of every
    ntype; `gather(gids)` returns the rows of arbitrary gids via owner bucketing (libgsb),
    NCCL all-to-all of ids, a shard gather on the owners (libgsb), an all-to-all of rows back
    and an unpack (libgsb).  Collectives are issued from the current stream."""

    def __init__(self, counts, world: int, rank: int, shards, dim: int, group=None):
        import ctypes as C
        import numpy as np
        from ._lib import call
        self.world, self.rank, self.group, self.dim = world, rank, group, dim
        self.counts = np.asarray(counts, dtype=np.int64)
        self.bounds = balanced_bounds(self.counts, world)
        h = C.c_void_p()
        call("gsb_partition_create", len(self.counts), self.counts.ctypes.data_as(C.c_void_p), world, rank,
             self.bounds.ctypes.data_as(C.c_void_p), C.byref(h))
        self.h = h
        self.shards = [s.contiguous() for s in shards]
        from .runtime import DTYPE_CODE
        self.dtype = self.shards[0].dtype
        self.esize = self.shards[0].element_size()
        for t, sh in enumerate(self.shards):
            call("gsb_partition_set_shard", self.h, t, C.c_void_p(sh.data_ptr()), dim, DTYPE_CODE[sh.dtype])
        dev = self.shards[0].device
        self.counts_dev = torch.zeros(world, dtype=torch.int64, device=dev)
        self.ws = torch.zeros(world, dtype=torch.int64, device=dev)
        self.bytes_sent = 0

    def __del__(self):
        try:
            from ._lib import lib
            lib().gsb_partition_destroy(self.h)
        except Exception:
            pass

    def gather(self, gids: torch.Tensor, n: int, out: Optional[torch.Tensor] = None,
               rows_out: Optional[torch.Tensor] = None, perm_out: Optional[torch.Tensor] = None):
        """Rows of gids[:n].  With `out`, unpacks into out (gid order) and returns it; without,
        returns (rows in exchange order, perm) so that row i of the request is rows[perm[i]]
        (the consumer reads through perm -- no unpack pass).  rows_out / perm_out: fixed
        buffers (>= n rows) to receive them, so a captured compute graph can read them."""
        import ctypes as C
        import torch.distributed as dist
        from ._lib import call
        P = lambda x: C.c_void_p(x.data_ptr())
        s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        dev = gids.device
        send_gid = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
        perm = perm_out if perm_out is not None else torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        call("gsb_bucket_by_owner", self.h, P(gids), None, n, P(send_gid), P(perm), P(self.counts_dev), P(self.ws), s)
        recv_counts = torch.empty_like(self.counts_dev)
        dist.all_to_all_single(recv_counts, self.counts_dev, group=self.group)          # C1
        both = torch.cat([self.counts_dev, recv_counts]).cpu().tolist()
        send_splits, recv_splits = both[:self.world], both[self.world:]
        recv_gid = torch.empty(sum(recv_splits), dtype=torch.int64, device=dev)
        dist.all_to_all_single(recv_gid, send_gid[:n], recv_splits, send_splits, group=self.group)   # C4
        rows = torch.empty((max(sum(recv_splits), 1), self.dim), dtype=self.dtype, device=dev)
        call("gsb_shard_gather", self.h, P(recv_gid), recv_gid.numel(), P(rows), s)
        back = rows_out if rows_out is not None else torch.empty((max(n, 1), self.dim), dtype=self.dtype, device=dev)
        dist.all_to_all_single(back[:n], rows[:sum(recv_splits)], send_splits, recv_splits, group=self.group)  # C5
        self.bytes_sent += (n - send_splits[self.rank]) * 8 + (sum(recv_splits) - recv_splits[self.rank]) * self.dim * self.esize
        if out is None:
            return back, perm
        call("gsb_rows_permute", P(back), self.dim * self.esize, P(perm), None, n, P(out), s)
        return out


class PeerFeatures:
    """Partitioned features read over NVLink (§8(e)): this rank allocates only its node-ID
    range of every ntype; the shards of all ranks are mapped into every process with CUDA IPC
    and registered in the graph store, so the fused layer-0 gather+aggregation (and
    gsb_gather) load each row straight from its owner's HBM.  No collective on the data path."""

    def __init__(self, store, counts, world: int, rank: int, shards, dim: int, group=None):
        import ctypes as C
        import numpy as np
        import torch.distributed as dist
        from ._lib import call
        from .runtime import DTYPE_CODE
        self.bounds = balanced_bounds(counts, world)
        self.shards = [s.contiguous() for s in shards]
        mine = []
        for sh in self.shards:
            if sh.numel() == 0:
                mine.append(None)
                continue
            h = (C.c_char * 64)()
            off = C.c_int64()
            call("gsb_ipc_handle", C.c_void_p(sh.data_ptr()), h, C.byref(off))
            mine.append((bytes(h), int(off.value)))
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        self.mapped = []
        for t in range(len(self.shards)):
            ptrs = (C.c_void_p * world)()
            for w in range(world):
                if w == rank:
                    ptrs[w] = self.shards[t].data_ptr() if self.shards[t].numel() else None
                elif allh[w][t] is None:
                    ptrs[w] = None
                else:
                    hb, off = allh[w][t]
                    p = C.c_void_p()
                    call("gsb_ipc_open", (C.c_char * 64).from_buffer_copy(hb), off, C.byref(p))
                    ptrs[w] = p.value
                    self.mapped.append(p.value - off)
            b = np.ascontiguousarray(self.bounds[t])
            call("gsb_graph_set_feature_peers", store.h, t, world, b.ctypes.data_as(C.c_void_p), ptrs,
                 int(self.shards[t].shape[1]) if self.shards[t].dim() == 2 else dim, DTYPE_CODE[self.shards[t].dtype])
        store.feat_dim = dim
        store.feat_dtype = self.shards[0].dtype
        self.store = store


class PeerCSC:
    """Node-ID partitioned topology read over NVLink (§8(e); "a
    worker reads only its own partition's storage"): rank w built (GraphStore.load_etype_range)
    the CSC of every etype over the dst nodes it owns; the shards of all ranks are mapped into
    every process with CUDA IPC and registered (gsb_graph_set_csc_peers), so the sampling
    kernels read each dst's in-edge segment from its owner's HBM.  Keyed draws make the blocks
    identical to the whole-graph sampler's (bit-exact), with no collective on the data path."""

    def __init__(self, store, world: int, rank: int, bounds, group=None, map_peers: bool = True):
        """map_peers=False: register the partition bounds and this rank's own shard only (the
        NCCL exchange mode, SampleExchange, never reads another rank's CSC)."""
        import ctypes as C
        import numpy as np
        import torch.distributed as dist
        from ._lib import call
        self.bounds = np.ascontiguousarray(bounds, dtype=np.int64)        # [T][world+1]
        if not map_peers:
            nb = C.c_size_t()
            call("gsb_csc_peers_bytes", C.byref(nb))
            self.table = torch.zeros(int(nb.value), dtype=torch.uint8, device=store.device)
            self.mapped = []
            s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
            for r in range(store.R):
                ip = (C.c_void_p * world)()
                ix = (C.c_void_p * world)()
                eb = (C.c_int64 * world)()
                for w in range(world):      # other ranks' entries: never dereferenced
                    ip[w] = store.indptr[r].data_ptr()
                    ix[w] = store.indices[r].data_ptr()
                    eb[w] = int(store.eid_base[r])
                tot = torch.tensor([store.n_edges[r]], dtype=torch.int64, device=store.device)
                dist.all_reduce(tot, group=group)
                call("gsb_graph_set_csc_peers", store.h, C.c_void_p(self.table.data_ptr()), r, world,
                     self.bounds.ctypes.data_as(C.c_void_p), ip, ix, eb, int(tot.item()), s)
            store._csc_peers = self
            return
        mine = []
        for r in range(store.R):
            hs = []
            for t in (store.indptr[r], store.indices[r]):
                h = (C.c_char * 64)()
                off = C.c_int64()
                call("gsb_ipc_handle", C.c_void_p(t.data_ptr()), h, C.byref(off))
                hs.append((bytes(h), int(off.value)))
            mine.append((hs, int(store.eid_base[r]), int(store.n_edges[r])))
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        nb = C.c_size_t()
        call("gsb_csc_peers_bytes", C.byref(nb))
        dev = store.device
        self.table = torch.zeros(int(nb.value), dtype=torch.uint8, device=dev)
        self.mapped = []
        s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        for r in range(store.R):
            ip = (C.c_void_p * world)()
            ix = (C.c_void_p * world)()
            eb = (C.c_int64 * world)()
            for w in range(world):
                (hip, hix), base, _ = allh[w][r]
                eb[w] = base
                if w == rank:
                    ip[w] = store.indptr[r].data_ptr()
                    ix[w] = store.indices[r].data_ptr()
                    continue
                for arr, (hb, off) in ((ip, hip), (ix, hix)):
                    p = C.c_void_p()
                    call("gsb_ipc_open", (C.c_char * 64).from_buffer_copy(hb), off, C.byref(p))
                    arr[w] = p.value
                    self.mapped.append(p.value - off)
            call("gsb_graph_set_csc_peers", store.h, C.c_void_p(self.table.data_ptr()), r, world,
                 self.bounds.ctypes.data_as(C.c_void_p), ip, ix, eb, sum(allh[w][r][2] for w in range(world)), s)
        store._csc_peers = self


class SampleExchange:
    """NCCL frontier exchange of the partitioned graph (§8(e) C2/C3 as north_star states it;
    P:L86): every rank holds only the CSC of the dst nodes it owns
    (GraphStore.load_etype_range + partition bounds registered through PeerCSC(..., map=False))
    and never reads another rank's storage.  For every hop >= first_hop, gsb_sample
    buckets the frontier by owner, this object's callback all-to-alls the requests (C2), the
    owners sample them with the keyed RNG, and the callback all-to-alls the per-(request, slot)
    counts and the sampled (src gid, eid) edges back (C3); gsb_sample unpacks them into frontier
    order.  Exact-size all-to-alls: the sizes are read on the host (two syncs per hop), so the
    sample phase runs eagerly (no CUDA graph) in this mode.  Buffers are torch tensors sized by
    gsb_exchange_sizes (worst-case capacities, no device allocation in the library)."""

    def __init__(self, sampler, world: int, rank: int, first_hop: int = 1, group=None):
        import ctypes as C
        from . import _lib
        from ._lib import call
        self.world, self.rank, self.group = world, rank, group
        self.S = max(len(x) for x in sampler.store.slot_etypes())
        vals = [C.c_int64() for _ in range(6)]
        call("gsb_exchange_sizes", sampler.h, world, *[C.byref(v) for v in vals])
        cap_dst, cap_recv, cap_srv_e, cap_resp_e, srv_cnt_len, meta_b = [int(v.value) for v in vals]
        dev = sampler.arena.device
        I64 = lambda n: torch.zeros(max(int(n), 1), dtype=torch.int64, device=dev)
        S = self.S
        self.req_send, self.req_perm = I64(cap_dst), torch.zeros(cap_dst, dtype=torch.int32, device=dev)
        self.send_cnt, self.cursor = I64(world), I64(world)
        self.req_recv, self.xoff = I64(cap_recv), I64(world + 1)
        self.srv_meta = torch.zeros(meta_b, dtype=torch.uint8, device=dev)
        self.srv_cnt, self.srv_seg = I64(srv_cnt_len), I64(cap_recv * S + 1)
        self.srv_gid, self.srv_eid, self.srv_wcnt = I64(cap_srv_e), I64(cap_srv_e), I64(world)
        self.resp_cnt, self.resp_seg = I64(cap_dst * S + 1), I64(cap_dst * S + 1)
        self.resp_gid, self.resp_eid = I64(cap_resp_e), I64(cap_resp_e)
        P = lambda t: C.c_void_p(t.data_ptr())
        b = _lib.gsb_exchange_bufs(P(self.req_send), P(self.req_perm), P(self.send_cnt), P(self.cursor),
                                   P(self.req_recv), cap_recv, P(self.xoff), P(self.srv_meta), P(self.srv_cnt),
                                   P(self.srv_seg), P(self.srv_gid), P(self.srv_eid), cap_srv_e, P(self.srv_wcnt),
                                   P(self.resp_cnt), P(self.resp_seg), P(self.resp_gid), P(self.resp_eid), cap_resp_e)
        self._bufs = b
        self._fn = _lib.EXCHANGE_FN(self._callback)     # kept alive with self
        self.bytes_sent = 0
        call("gsb_blocks_set_exchange", sampler.h, world, rank, first_hop, C.byref(b), self._fn, None)
        self.sampler = sampler
        self.first_hop = first_hop
        self.host_s = {}                # host seconds spent in the callback, per phase (tools)
        sampler._sx = self              # kept alive with the sampler; twin() attaches its own

    def _a2a(self, out, inp, out_splits, in_splits):
        import torch.distributed as dist
        dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)

    def _callback(self, user, phase, hop, stream, counts):
        import time
        t0 = time.perf_counter()
        try:
            return self._callback_body(phase, stream, counts)
        finally:
            self.host_s[phase] = self.host_s.get(phase, 0.0) + time.perf_counter() - t0

    def _callback_body(self, phase, stream, counts):
        try:
            st = torch.cuda.ExternalStream(stream) if stream else torch.cuda.default_stream()
            with torch.cuda.stream(st):
                w = self.world
                if phase == 0:
                    recv = torch.empty_like(self.send_cnt)
                    self._a2a(recv, self.send_cnt, None, None)                       # C1: counts
                    both = torch.cat([self.send_cnt, recv]).tolist()                 # host sync
                    self.sc, self.rc = both[:w], both[w:]
                    ns, nr = sum(self.sc), sum(self.rc)
                    self._a2a(self.req_recv[:nr], self.req_send[:ns], self.rc, self.sc)   # C2: request ids
                    for k in range(w):
                        counts[k] = self.rc[k]
                    self.bytes_sent += (ns - self.sc[self.rank]) * 8
                    return 0
                S = self.S
                er_t = torch.empty_like(self.srv_wcnt)
                self._a2a(er_t, self.srv_wcnt, None, None)                          # edge counts
                both = torch.cat([self.srv_wcnt, er_t]).tolist()                     # one host sync
                ew, er = both[:w], both[w:]
                ns, nr = sum(self.sc), sum(self.rc)
                self._a2a(self.resp_cnt[:ns * S], self.srv_cnt[:nr * S], [x * S for x in self.sc],
                          [x * S for x in self.rc])                                  # C3: counts
                self._a2a(self.resp_gid[:sum(er)], self.srv_gid[:sum(ew)], er, ew)   # C3: edges
                self._a2a(self.resp_eid[:sum(er)], self.srv_eid[:sum(ew)], er, ew)
                self.bytes_sent += (nr - self.rc[self.rank]) * S * 8 + (sum(ew) - ew[self.rank]) * 16
                return 0
        except Exception as e:   # reported through the library's status
            import sys
            print(f"[gsb] exchange callback failed: {e!r}", file=sys.stderr)
            return 1


class PeerEmbedding:
    """A learnable table (§8(f) f1) partitioned over the ranks of one box (R-sparsedist): rank
    w holds rows [bounds[w], bounds[w+1]) of the table, its Adagrad state, a gradient
    accumulator and a touched bitmap; the table, accumulator and bitmap shards of every rank
    are mapped into every process with CUDA IPC.  Forward loads each input row from its owner
    (gsb_sparse_emb_fwd_peers); the update pushes 1/world of every touched dH0 row into the
    owner's accumulator (gsb_sparse_emb_push), then -- after a barrier -- every owner takes one
    Adagrad step per touched row (gsb_sparse_adagrad_apply); a second barrier orders the
    update before the next forward.  The barriers are 1-element NCCL all-reduces on the
    compute stream (device-side ordering, no host sync)."""

    def __init__(self, E_full, world: int, rank: int, group=None):
        import ctypes as C
        import numpy as np
        import torch
        import torch.distributed as dist
        from ._lib import call
        n, d = int(E_full.shape[0]), int(E_full.shape[1])
        self.world, self.rank, self.group, self.d = world, rank, group, d
        self.bounds = np.array([n * w // world for w in range(world + 1)], np.int64)
        lo, hi = int(self.bounds[rank]), int(self.bounds[rank + 1])
        dev = torch.device("cuda", torch.cuda.current_device())
        rows = max(hi - lo, 1)
        self.E = torch.zeros((rows, d), dtype=torch.float32, device=dev)
        self.E[: hi - lo].copy_(E_full[lo:hi])
        self.state = torch.zeros_like(self.E)
        self.G = torch.zeros_like(self.E)
        self.bits = torch.zeros((rows + 31) // 32, dtype=torch.int32, device=dev)
        self.n_rows = hi - lo
        self.tok = torch.zeros(1, dtype=torch.float32, device=dev)
        mine = []
        for t in (self.E, self.G, self.bits):
            h = (C.c_char * 64)()
            off = C.c_int64()
            call("gsb_ipc_handle", C.c_void_p(t.data_ptr()), h, C.byref(off))
            mine.append((bytes(h), int(off.value)))
        allh = [None] * world
        dist.all_gather_object(allh, mine, group=group)
        self.ptrs = []
        self.mapped = []
        for k, own in enumerate((self.E, self.G, self.bits)):
            arr = (C.c_void_p * world)()
            for w in range(world):
                if w == rank:
                    arr[w] = own.data_ptr()
                else:
                    hb, off = allh[w][k]
                    p = C.c_void_p()
                    call("gsb_ipc_open", (C.c_char * 64).from_buffer_copy(hb), off, C.byref(p))
                    arr[w] = p.value
                    self.mapped.append(p.value - off)
            self.ptrs.append(arr)
        self._bnd = self.bounds.ctypes.data_as(C.c_void_p)

    def barrier(self):
        import torch.distributed as dist
        dist.all_reduce(self.tok, group=self.group)

    def fwd(self, sampler, ntype: int, H0, stream):
        import ctypes as C
        from ._lib import call
        call("gsb_sparse_emb_fwd_peers", sampler.h, C.c_void_p(sampler.arena.data_ptr()), ntype, self.world,
             self._bnd, self.ptrs[0], self.d, C.c_void_p(H0.data_ptr()), stream)

    def push(self, sampler, ntype: int, dH0, stream):
        import ctypes as C
        from ._lib import call
        call("gsb_sparse_emb_push", sampler.h, C.c_void_p(sampler.arena.data_ptr()), ntype, self.world, self._bnd,
             self.ptrs[1], self.ptrs[2], C.c_void_p(dH0.data_ptr()), self.d, 1.0 / self.world, stream)

    def apply(self, lr: float, eps: float, stream):
        import ctypes as C
        from ._lib import call
        call("gsb_sparse_adagrad_apply", C.c_void_p(self.E.data_ptr()), C.c_void_p(self.state.data_ptr()),
             C.c_void_p(self.G.data_ptr()), C.c_void_p(self.bits.data_ptr()), self.n_rows, self.d, lr, eps, stream)

    def update(self, sampler, ntype: int, dH0, lr: float, eps: float, stream, pushed: bool = False):
        """push -> barrier -> apply -> barrier.  pushed: the push was issued before a collective
        that already separates it from the apply (the dense-gradient all-reduce)."""
        if not pushed:
            self.push(sampler, ntype, dH0, stream)
            self.barrier()
        self.apply(lr, eps, stream)
        self.barrier()

    def gather_full(self):
        """The whole table (all shards) on every rank, for checks: NCCL all-gather."""
        import torch
        import torch.distributed as dist
        parts = [torch.zeros((max(int(self.bounds[w + 1] - self.bounds[w]), 1), self.d), device=self.E.device)
                 for w in range(self.world)]
        dist.all_gather(parts, self.E, group=self.group)
        return torch.cat([p[: int(self.bounds[w + 1] - self.bounds[w])] for w, p in enumerate(parts)])
