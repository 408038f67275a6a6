// gsb_internal.cuh -- shared internals of libgsb (CUDA path).  Independent of oracle/.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <algorithm>
#include <utility>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/gsb.h"

namespace gsb {

constexpr int kMaxT = GSB_MAX_NTYPES;
constexpr int kMaxR = GSB_MAX_ETYPES;
constexpr int kMaxS = GSB_MAX_SLOTS;
constexpr int kMaxL = GSB_MAX_LAYERS;
constexpr int kNumSMs = 148;  // B200
constexpr int kMaxPeers = 8;  // GPUs of one NVSwitch box

// ------------------------------------------------------------------------------------
// errors / instrumentation
// ------------------------------------------------------------------------------------
void set_error(const char* fmt, ...);
gsb_status cuda_status(cudaError_t e, const char* what);
void prof_begin(const char* name, cudaStream_t s);
void prof_end(cudaStream_t s);
void count_launch(int n = 1);

#define GSB_CHECK_ARG(cond, ...)           \
    do {                                   \
        if (!(cond)) {                     \
            ::gsb::set_error(__VA_ARGS__); \
            return GSB_EINVAL;             \
        }                                  \
    } while (0)

#define GSB_CUDA(call)                                                \
    do {                                                              \
        cudaError_t _e = (call);                                      \
        if (_e != cudaSuccess) return ::gsb::cuda_status(_e, #call); \
    } while (0)

// Programmatic dependent launch (PDL, opt-in with GSB_PDL=1): every libgsb kernel can be
// launched with programmatic stream serialization, so its grid is set up while its
// predecessor in the stream drains (also inside CUDA graphs); each kernel starts with
// GSB_PDL_ENTRY: wait for the predecessor grid's completion and memory (before any read or
// write), then let its own dependent launch early.  Off by default: under the step's CUDA
// graphs it measured between +0.9 % and -3.7 % (the parity suite passes either way).  Without
// the attribute the waits are no-ops.
bool pdl_enabled();
#define GSB_PDL_ENTRY()                                            \
    do {                                                           \
        asm volatile("griddepcontrol.wait;" ::: "memory");         \
        asm volatile("griddepcontrol.launch_dependents;" :::);     \
    } while (0)

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Launch with instrumentation: counts the launch, optionally brackets it with events.
#define GSB_LAUNCH(name, kern, grid, block, smem, stream, ...)                        \
    do {                                                                              \
        ::gsb::prof_begin(name, stream);                                              \
        cudaError_t _e = ::gsb::launch_k(kern, dim3(grid), dim3(block), (size_t)(smem), \
                                         (cudaStream_t)(stream), __VA_ARGS__);       \
        ::gsb::prof_end(stream);                                                      \
        ::gsb::count_launch();                                                        \
        if (_e == cudaSuccess) _e = cudaGetLastError();                               \
        if (_e != cudaSuccess) return ::gsb::cuda_status(_e, name);                   \
    } while (0)

// ------------------------------------------------------------------------------------
// Fork / join onto a library-owned side stream (one per device), so independent kernels of
// one call (e.g. a weight gradient and the input gradient) overlap.  Works inside CUDA graph
// capture: the side stream joins the capture through the fork event and is joined back
// before the call returns.  fork_begin returns the side stream (or s itself when forking is
// disabled with GSB_NO_FORK=1).
// ------------------------------------------------------------------------------------
cudaStream_t fork_begin(cudaStream_t s);
gsb_status fork_end(cudaStream_t s, cudaStream_t side);

// ------------------------------------------------------------------------------------
// graph descriptor passed to kernels by value
// ------------------------------------------------------------------------------------
struct GraphDev {
    int32_t T, R, S;                    // ntypes, etypes, max slots
    int32_t feat_dim;                   // elements per feature row when uniform over ntypes, else 0
    int32_t feat_dtype;                 // GSB_F32 / GSB_BF16 (one element type for all ntypes)
    int32_t feat_row_bytes;             // feat_dim * element size (uniform case)
    int32_t dim_t[kMaxT];               // per-ntype row width (elements; 0 = not registered)
    int32_t row_bytes_t[kMaxT];         // per-ntype row bytes (multiple of 16)
    int64_t node_off[kMaxT + 1];
    int32_t src_t[kMaxR], dst_t[kMaxR];
    int32_t n_slots[kMaxT];             // in-relations of each ntype
    int32_t slot_etype[kMaxT][kMaxS];   // etype of slot s of ntype t
    const int64_t* indptr[kMaxR];
    const int32_t* indices[kMaxR];
    int64_t eid_base[kMaxR];
    const char* feat[kMaxT];
    // node-ID partitioned features read over NVLink (peer.cu): rank w owns local ids
    // [plo[t][w], plo[t][w+1]) of ntype t at peer[t][w] (an IPC-mapped pointer for w != self)
    int32_t nparts;
    int64_t plo[kMaxT][kMaxPeers + 1];
    const char* peer[kMaxT][kMaxPeers];
    // node-ID partitioned topology (peer.cu, §8(e)): device table of every rank's CSC shard,
    // or null when this process holds the whole CSC (indptr / indices above)
    const struct CscPeers* cpeers;
};

// Partitioned CSC: rank w holds the in-edges of the dst nodes it owns, local ids
// [lo[t][w], lo[t][w+1]) of every ntype t, as a CSC over that range (positions local to its
// own indices array) whose first edge has global CSC position eid_base[r][w].  Segments of
// other ranks' dst nodes are read from the owner's HBM over NVLink (CUDA IPC pointers).
// Lives in caller-owned device memory (gsb_csc_peers_bytes).
struct CscPeers {
    int32_t world;
    int64_t lo[kMaxT][kMaxPeers + 1];
    const int64_t* indptr[kMaxR][kMaxPeers];
    const int32_t* indices[kMaxR][kMaxPeers];
    int64_t eid_base[kMaxR][kMaxPeers];
};

// In-edge segment of dst local id vl (ntype t) in etype r: indices seg[0..deg), edge ids
// eid0 + position.  Whole CSC, or the owner's shard of a partitioned one.
struct CscSeg {
    const int32_t* seg;
    int64_t deg, eid0;
};
__device__ __forceinline__ CscSeg csc_seg(const GraphDev& g, int r, int t, int64_t vl) {
    CscSeg c;
    if (g.cpeers) {
        const CscPeers& P = *g.cpeers;
        int w = 0;
#pragma unroll 1
        for (int k = 1; k < P.world; ++k) w += (vl >= P.lo[t][k]) ? 1 : 0;
        const int64_t* ip = P.indptr[r][w] + (vl - P.lo[t][w]);
        const int64_t a = ip[0];
        c.deg = ip[1] - a;
        c.seg = P.indices[r][w] + a;
        c.eid0 = P.eid_base[r][w] + a;
    } else {
        const int64_t a = g.indptr[r][vl];
        c.deg = g.indptr[r][vl + 1] - a;
        c.seg = g.indices[r] + a;
        c.eid0 = g.eid_base[r] + a;
    }
    return c;
}

__host__ __device__ inline int type_of(const GraphDev& g, int64_t gid) {
    int t = 0;
#pragma unroll 1
    for (int k = 1; k < g.T; ++k) t += (gid >= g.node_off[k]) ? 1 : 0;
    return t;
}

// Row of node gid in its feature table (16-byte chunks): local table, or the owner's
// (possibly peer) shard.
__device__ __forceinline__ const uint4* feat_row(const GraphDev& g, int64_t gid) {
    const int t = type_of(g, gid);
    const int64_t local = gid - g.node_off[t];
    if (g.nparts > 1) {
        int w = 0;
#pragma unroll 1
        for (int k = 1; k < g.nparts; ++k) w += (local >= g.plo[t][k]) ? 1 : 0;
        return reinterpret_cast<const uint4*>(g.peer[t][w] + (local - g.plo[t][w]) * g.row_bytes_t[t]);
    }
    return reinterpret_cast<const uint4*>(g.feat[t] + local * g.row_bytes_t[t]);
}

inline int dtype_size(int32_t dtype) { return dtype == GSB_BF16 ? 2 : (dtype == GSB_F32 ? 4 : 0); }

struct Graph;
// feature row format shared by all ntypes (core.cu)
gsb_status set_feature_format(Graph* G, int32_t ntype, int32_t dim, int32_t dtype);
gsb_status launch_gather(const Graph* G, const int64_t* gid, const int64_t* n_dev, int64_t n_host, int64_t n_max,
                         void* out, cudaStream_t s);

// Per-hop sizes, written by kernels (device resident; never copied to the host on the
// hot path).  dst rows of ntype t are [dst_off[t], dst_off[t+1]); src rows likewise.
struct HopMeta {
    int64_t n_dst;
    int64_t n_edges;
    int64_t n_src;
    int64_t dst_off[kMaxT + 1];
    int64_t src_off[kMaxT + 1];
    int64_t new_base[kMaxT];   // bitmap rank of node_off[t] (first new node of type t)
};

// Per-hop device buffers inside the arena.
struct HopBufs {
    int64_t cap_dst, cap_edges, cap_src;
    int64_t cap_seeds;    // the batch's seed capacity (hop 1's cap_dst): a host-side size hint
    HopMeta* meta;
    int64_t* dst_gid;     // [cap_dst]   (hop 1: seed copy; else previous hop's src_gid)
    int64_t* cnt;         // [cap_dst*S + 1]
    int64_t* seg_ptr;     // [cap_dst*S + 1]
    int64_t* e_src_gid;   // [cap_edges]
    int64_t* e_eid;       // [cap_edges]
    int32_t* e_src;       // [cap_edges]
    int64_t* src_gid;     // [cap_src]
    CscSeg* segc;         // [cap_dst*S] the (dst, slot) segments count resolved, reused by fill
    // by-source transposed CSR of the block (§8(a) a4; hops feeding layers >= 1, else null):
    // the edges of src row u are t_edge[t_ptr[u] .. t_ptr[u+1]) in ascending edge order;
    // e_seg[e] = (dst row, slot) segment of edge e
    int32_t* e_seg;       // [cap_edges]
    int32_t* t_key;       // [cap_edges] sort keys (src row; past the live edges INT32_MAX); after the
                          //   sort: t_seg, the segment id of transposed position k
    int32_t* t_key2;      // [cap_edges]
    int32_t* t_val;       // [cap_edges] edge ids before the sort; after it: 1 / segment count (fp32 bits)
    int32_t* t_edge;      // [cap_edges]
    int32_t* t_ptr;       // [cap_src + 1]
};

struct Graph {
    GraphDev dev;
    CscPeers* cpeers_host = nullptr;   // host mirror of the partitioned-CSC table (peer.cu)
    bool dtype_set = false;
    int64_t counts[kMaxT];
    int64_t n_edges[kMaxR];
    int64_t total_nodes;
};

// NCCL exchange of the sampling frontier (§8(e) C2/C3; gsb_blocks_set_exchange): caller-owned
// device buffers; all zero = off.
struct Xchg {
    int32_t world, rank, first_hop;                 // first_hop 0: exchange off
    int64_t* req_send;   // [cap_dst] frontier gids grouped by owner
    int32_t* req_perm;   // [cap_dst] position of frontier row j in req_send
    int64_t* send_cnt;   // [world] requests per owner (device; read by the callback)
    int64_t* cursor;     // [world]
    int64_t* req_recv;   // [cap_recv] requests received, grouped by requesting rank
    int64_t cap_recv;
    int64_t* xoff;       // [world+1] prefix of the received request counts (device)
    HopMeta* srv_meta;   // n_dst = received requests
    int64_t* srv_cnt;    // [cap_recv*S + 1 + kCntMaxBlocks] per (request, slot) counts
    int64_t* srv_seg;    // [cap_recv*S + 1]
    int64_t* srv_gid;    // [cap_srv_e] sampled edges of the served requests
    int64_t* srv_eid;
    int64_t cap_srv_e;
    int64_t* srv_wcnt;   // [world] edges to return to each requesting rank (device)
    int64_t* resp_cnt;   // [cap_dst*S + 1] counts of this rank's requests, in req_send order
    int64_t* resp_seg;   // [cap_dst*S + 1]
    int64_t* resp_gid;   // [cap_resp_e] returned edges, grouped by owner in req_send order
    int64_t* resp_eid;
    int64_t cap_resp_e;
    gsb_exchange_fn fn;
    void* user;
};

struct Blocks {
    Graph* g;
    Xchg x;
    int32_t L;
    int32_t fanout[kMaxL];     // f[l] for layer l
    int64_t max_seeds, max_excl;
    // arena layout (byte offsets)
    size_t off_meta[kMaxL + 1];
    size_t off_seed, off_cnt[kMaxL], off_seg[kMaxL], off_esrcgid[kMaxL], off_eeid[kMaxL], off_esrc[kMaxL];
    size_t off_src[kMaxL], off_segc[kMaxL];
    size_t off_tcsr[kMaxL];   // transposed CSR block of hop h (0: none)
    size_t off_map, off_bitmap, off_wrank, off_err, off_cub, off_excl;
    size_t cub_bytes, total_bytes;
    int64_t cap_dst[kMaxL + 1], cap_edges[kMaxL];
    int64_t n_words;
    HopBufs hop(int h, void* arena) const;   // h = 1..L
    int hop_of_layer(int layer) const { return L - layer; }
};

template <typename T>
inline T* at(void* base, size_t off) {
    return reinterpret_cast<T*>(static_cast<char*>(base) + off);
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

inline int grid_for(int64_t work, int per_block, int max_blocks = kNumSMs * 16) {
    int64_t b = ceil_div(work, per_block);
    if (b < 1) b = 1;
    if (b > max_blocks) b = max_blocks;
    return (int)b;
}

// ------------------------------------------------------------------------------------
// device helpers
// ------------------------------------------------------------------------------------
__device__ __forceinline__ float4 ldg_nc_f4(const float4* p) {
    float4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ uint4 ldg_nc_u4(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// 16-byte chunk -> fp32 values: 4 floats (fp32 rows) or 8 bf16 widened exactly
template <bool BF16>
struct Chunk {
    static constexpr int kVec = BF16 ? 8 : 4;
};
__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

template <bool BF16>
__device__ __forceinline__ void chunk_acc(float* acc, const uint4 x) {
    if (BF16) {
        acc[0] += bf16_lo(x.x); acc[1] += bf16_hi(x.x); acc[2] += bf16_lo(x.y); acc[3] += bf16_hi(x.y);
        acc[4] += bf16_lo(x.z); acc[5] += bf16_hi(x.z); acc[6] += bf16_lo(x.w); acc[7] += bf16_hi(x.w);
    } else {
        acc[0] += __uint_as_float(x.x); acc[1] += __uint_as_float(x.y);
        acc[2] += __uint_as_float(x.z); acc[3] += __uint_as_float(x.w);
    }
}

// Warp-cooperative search in a non-decreasing offset array: the last i in [lo, hi) with
// ptr[i] <= a, given ptr[lo] <= a < ptr[hi]; 32 probes per round (log32 rounds).  Used to cut
// long (fanout ALL / full-CSC) segments into fixed-size edge pieces: the warp owning piece
// [a, b) finds the segments holding its first and last edge.
__device__ __forceinline__ int64_t seg_find(const int64_t* __restrict__ ptr, int64_t lo, int64_t hi, int64_t a,
                                            int lane) {
    while (hi - lo > 1) {
        const int64_t step = (hi - lo + 31) / 32;
        const int64_t p = lo + (int64_t)(lane + 1) * step;
        const bool le = p < hi && ptr[p] <= a;
        const int k = __popc(__ballot_sync(0xffffffffu, le));
        lo += (int64_t)k * step;
        hi = min(hi, lo + step);
    }
    return lo;
}

__device__ __forceinline__ void red_add_f4(float* p, float4 v) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w)
                 : "memory");
}

__device__ __forceinline__ void red_add_f1(float* p, float v) { atomicAdd(p, v); }

}  // namespace gsb
