// sparse_emb.cu -- learnable embedding tables for featureless node types (
// P:L156 "GraphStorm by default adds learnable embeddings on author nodes"): the layer-0
// input rows of such an ntype read the table, and after the backward pass only the rows the
// mini-batch touched are updated with sparse Adagrad (R-sparseopt).
// Contract: include/gsb.h "Learnable sparse embeddings".
#include "gsb_internal.cuh"

namespace gsb {

// thread per 16-byte chunk of an input row of type t:  H0[row] = E[gid - node_off[t]]
__global__ void emb_fwd_kernel(const HopMeta* __restrict__ m, const int64_t* __restrict__ src_gid, int t,
                               int64_t node_off_t, const float* __restrict__ E, int d, float* __restrict__ H0) {
    GSB_PDL_ENTRY();
    const int c4 = d >> 2;
    const int64_t r0 = m->src_off[t], n = (m->src_off[t + 1] - r0) * c4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = r0 + i / c4;
        const int c = (int)(i % c4);
        const int64_t local = __ldg(src_gid + row) - node_off_t;
        reinterpret_cast<float4*>(H0 + row * d)[c] = __ldg(reinterpret_cast<const float4*>(E + local * d) + c);
    }
}

// thread per 16-byte chunk of a touched row: state += g^2 ; E -= lr g / (sqrt(state) + eps)
// (rows of one ntype in a block's input list are distinct: no two threads share an element)
__global__ void emb_adagrad_kernel(const HopMeta* __restrict__ m, const int64_t* __restrict__ src_gid, int t,
                                   int64_t node_off_t, float* __restrict__ E, float* __restrict__ state,
                                   const float* __restrict__ dH0, int d, float lr, float eps) {
    GSB_PDL_ENTRY();
    const int c4 = d >> 2;
    const int64_t r0 = m->src_off[t], n = (m->src_off[t + 1] - r0) * c4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = r0 + i / c4;
        const int c = (int)(i % c4);
        const int64_t local = __ldg(src_gid + row) - node_off_t;
        const float4 g = __ldg(reinterpret_cast<const float4*>(dH0 + row * d) + c);
        float4* sp = reinterpret_cast<float4*>(state + local * d) + c;
        float4* ep = reinterpret_cast<float4*>(E + local * d) + c;
        float4 s = *sp, e = *ep;
        s.x += g.x * g.x; s.y += g.y * g.y; s.z += g.z * g.z; s.w += g.w * g.w;
        e.x -= lr * g.x / (sqrtf(s.x) + eps);
        e.y -= lr * g.y / (sqrtf(s.y) + eps);
        e.z -= lr * g.z / (sqrtf(s.z) + eps);
        e.w -= lr * g.w / (sqrtf(s.w) + eps);
        *sp = s;
        *ep = e;
    }
}

// ------------------------------------------------------------------------------------
// Tables partitioned over the GPUs of one NVSwitch box (§8(e) + §8(f) f1, R-sparsedist): rank
// w owns local rows [lo[w], lo[w+1]) of the table and its Adagrad state, plus a gradient
// accumulator G_w (zero between steps) and a touched bitmap; peers' shards are IPC-mapped.
//   fwd:   H0[i] = E_{owner}[x - lo[owner]]                          (NVLink loads)
//   push:  G_{owner}[x - lo] += scale * dH0[i]; set bit x - lo        (NVLink red.add.v4 / atomicOr)
//   apply: owner, every set bit: Adagrad with G row, then zero G row and the bit
// push and apply are separated by a cross-rank barrier (caller), as are apply and the next fwd.
// ------------------------------------------------------------------------------------
struct EmbPeers {
    int world;
    int64_t lo[kMaxPeers + 1];
    float* E[kMaxPeers];
    float* G[kMaxPeers];
    uint32_t* bits[kMaxPeers];
};

__device__ __forceinline__ int emb_owner(const EmbPeers& P, int64_t x) {
    int w = 0;
#pragma unroll 1
    for (int k = 1; k < P.world; ++k) w += (x >= P.lo[k]) ? 1 : 0;
    return w;
}

__global__ void emb_fwd_peers_kernel(const HopMeta* __restrict__ m, const int64_t* __restrict__ src_gid, int t,
                                     int64_t node_off_t, EmbPeers P, int d, float* __restrict__ H0) {
    GSB_PDL_ENTRY();
    const int c4 = d >> 2;
    const int64_t r0 = m->src_off[t], n = (m->src_off[t + 1] - r0) * c4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = r0 + i / c4;
        const int c = (int)(i % c4);
        const int64_t x = __ldg(src_gid + row) - node_off_t;
        const int w = emb_owner(P, x);
        reinterpret_cast<float4*>(H0 + row * d)[c] = reinterpret_cast<const float4*>(P.E[w] + (x - P.lo[w]) * d)[c];
    }
}

__global__ void emb_push_kernel(const HopMeta* __restrict__ m, const int64_t* __restrict__ src_gid, int t,
                                int64_t node_off_t, EmbPeers P, const float* __restrict__ dH0, int d, float scale) {
    GSB_PDL_ENTRY();
    const int c4 = d >> 2;
    const int64_t r0 = m->src_off[t], n = (m->src_off[t + 1] - r0) * c4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = r0 + i / c4;
        const int c = (int)(i % c4);
        const int64_t x = __ldg(src_gid + row) - node_off_t;
        const int w = emb_owner(P, x);
        const int64_t l = x - P.lo[w];
        const float4 g = __ldg(reinterpret_cast<const float4*>(dH0 + row * d) + c);
        red_add_f4(P.G[w] + l * d + 4 * c, make_float4(scale * g.x, scale * g.y, scale * g.z, scale * g.w));
        if (c == 0) atomicOr(P.bits[w] + (l >> 5), 1u << (l & 31));
    }
}

// warp per 32-row bitmap word; lanes over the 16-byte chunks of each set row
__global__ void __launch_bounds__(256) emb_apply_kernel(float* __restrict__ E, float* __restrict__ state,
                                                        float* __restrict__ G, uint32_t* __restrict__ bits,
                                                        int64_t n_rows, int d, float lr, float eps) {
    GSB_PDL_ENTRY();
    const int lane = threadIdx.x & 31;
    const int c4 = d >> 2;
    const int64_t n_words = (n_rows + 31) >> 5;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t wd = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; wd < n_words; wd += warps) {
        uint32_t b = bits[wd];
        if (!b) continue;
        if (lane == 0) bits[wd] = 0u;
        while (b) {
            const int k = __ffs(b) - 1;
            b &= b - 1;
            const int64_t l = wd * 32 + k;
            for (int c = lane; c < c4; c += 32) {
                float4* gp = reinterpret_cast<float4*>(G + l * d) + c;
                float4* sp = reinterpret_cast<float4*>(state + l * d) + c;
                float4* ep = reinterpret_cast<float4*>(E + l * d) + c;
                const float4 g = *gp;
                float4 s = *sp, e = *ep;
                s.x += g.x * g.x; s.y += g.y * g.y; s.z += g.z * g.z; s.w += g.w * g.w;
                e.x -= lr * g.x / (sqrtf(s.x) + eps);
                e.y -= lr * g.y / (sqrtf(s.y) + eps);
                e.z -= lr * g.z / (sqrtf(s.z) + eps);
                e.w -= lr * g.w / (sqrtf(s.w) + eps);
                *sp = s;
                *ep = e;
                *gp = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
    }
}

static gsb_status emb_peers(int32_t world, const int64_t* bounds, void* const* E, void* const* G, void* const* bits,
                            EmbPeers& P) {
    GSB_CHECK_ARG(world >= 1 && world <= kMaxPeers && bounds, "world %d (1..%d) / bounds", world, kMaxPeers);
    P = EmbPeers{};
    P.world = world;
    for (int w = 0; w <= world; ++w) P.lo[w] = bounds[w];
    GSB_CHECK_ARG(bounds[0] == 0, "bounds[0] must be 0");
    for (int w = 0; w < world; ++w) {
        GSB_CHECK_ARG(bounds[w + 1] >= bounds[w], "bounds not monotone");
        if (E) { GSB_CHECK_ARG(E[w], "null shard %d", w); P.E[w] = static_cast<float*>(E[w]); }
        if (G) { GSB_CHECK_ARG(G[w] && bits && bits[w], "null accumulator %d", w); P.G[w] = static_cast<float*>(G[w]);
                 P.bits[w] = static_cast<uint32_t*>(bits[w]); }
    }
    return GSB_OK;
}

static gsb_status emb_args(Blocks* B, const void* arena, int32_t ntype, int32_t d) {
    GSB_CHECK_ARG(B && arena, "null argument");
    GSB_CHECK_ARG(ntype >= 0 && ntype < B->g->dev.T, "ntype %d out of range", ntype);
    GSB_CHECK_ARG(d > 0 && d % 4 == 0, "d %d must be a multiple of 4", d);
    return GSB_OK;
}

}  // namespace gsb

using namespace gsb;

extern "C" {

gsb_status gsb_sparse_emb_fwd(gsb_blocks_t b, const void* arena, int32_t ntype, const float* E, int32_t d, float* H0,
                              void* stream) {
    Blocks* B = reinterpret_cast<Blocks*>(b);
    gsb_status st = emb_args(B, arena, ntype, d);
    if (st != GSB_OK) return st;
    GSB_CHECK_ARG(E && H0, "null table / H0");
    HopBufs hb = B->hop(B->L, const_cast<void*>(arena));
    GSB_LAUNCH("emb_fwd", emb_fwd_kernel, grid_for(hb.cap_src * (d / 4), 256, kNumSMs * 8), 256, 0,
               (cudaStream_t)stream, hb.meta, hb.src_gid, ntype, B->g->dev.node_off[ntype], E, d, H0);
    return GSB_OK;
}

gsb_status gsb_sparse_adagrad(gsb_blocks_t b, const void* arena, int32_t ntype, float* E, float* state,
                              const float* dH0, int32_t d, float lr, float eps, void* stream) {
    Blocks* B = reinterpret_cast<Blocks*>(b);
    gsb_status st = emb_args(B, arena, ntype, d);
    if (st != GSB_OK) return st;
    GSB_CHECK_ARG(E && state && dH0, "null table / state / dH0");
    HopBufs hb = B->hop(B->L, const_cast<void*>(arena));
    GSB_LAUNCH("emb_adagrad", emb_adagrad_kernel, grid_for(hb.cap_src * (d / 4), 256, kNumSMs * 8), 256, 0,
               (cudaStream_t)stream, hb.meta, hb.src_gid, ntype, B->g->dev.node_off[ntype], E, state, dH0, d, lr,
               eps);
    return GSB_OK;
}

gsb_status gsb_sparse_emb_fwd_peers(gsb_blocks_t b, const void* arena, int32_t ntype, int32_t world,
                                    const int64_t* bounds, void* const* E, int32_t d, float* H0, void* stream) {
    Blocks* B = reinterpret_cast<Blocks*>(b);
    gsb_status st = emb_args(B, arena, ntype, d);
    if (st != GSB_OK) return st;
    GSB_CHECK_ARG(E && H0, "null tables / H0");
    EmbPeers P;
    st = emb_peers(world, bounds, E, nullptr, nullptr, P);
    if (st != GSB_OK) return st;
    GSB_CHECK_ARG(bounds[world] == B->g->counts[ntype], "bounds[world] %lld != count of ntype %d",
                  (long long)bounds[world], ntype);
    HopBufs hb = B->hop(B->L, const_cast<void*>(arena));
    GSB_LAUNCH("emb_fwd", emb_fwd_peers_kernel, grid_for(hb.cap_src * (d / 4), 256, kNumSMs * 8), 256, 0,
               (cudaStream_t)stream, hb.meta, hb.src_gid, ntype, B->g->dev.node_off[ntype], P, d, H0);
    return GSB_OK;
}

gsb_status gsb_sparse_emb_push(gsb_blocks_t b, const void* arena, int32_t ntype, int32_t world, const int64_t* bounds,
                               void* const* G, void* const* touched, const float* dH0, int32_t d, float scale,
                               void* stream) {
    Blocks* B = reinterpret_cast<Blocks*>(b);
    gsb_status st = emb_args(B, arena, ntype, d);
    if (st != GSB_OK) return st;
    GSB_CHECK_ARG(G && touched && dH0, "null accumulators / bitmaps / dH0");
    EmbPeers P;
    st = emb_peers(world, bounds, nullptr, G, touched, P);
    if (st != GSB_OK) return st;
    GSB_CHECK_ARG(bounds[world] == B->g->counts[ntype], "bounds[world] %lld != count of ntype %d",
                  (long long)bounds[world], ntype);
    HopBufs hb = B->hop(B->L, const_cast<void*>(arena));
    GSB_LAUNCH("emb_push", emb_push_kernel, grid_for(hb.cap_src * (d / 4), 256, kNumSMs * 8), 256, 0,
               (cudaStream_t)stream, hb.meta, hb.src_gid, ntype, B->g->dev.node_off[ntype], P, dH0, d, scale);
    return GSB_OK;
}

gsb_status gsb_sparse_adagrad_apply(float* E, float* state, float* G, uint32_t* touched, int64_t n_rows, int32_t d,
                                    float lr, float eps, void* stream) {
    GSB_CHECK_ARG(n_rows >= 0 && d > 0 && d % 4 == 0, "n_rows %lld, d %d (multiple of 4)", (long long)n_rows, d);
    if (n_rows == 0) return GSB_OK;
    GSB_CHECK_ARG(E && state && G && touched, "null argument");
    GSB_LAUNCH("emb_apply", emb_apply_kernel, grid_for(((n_rows + 31) / 32) * 32, 256, kNumSMs * 8), 256, 0,
               (cudaStream_t)stream, E, state, G, touched, n_rows, d, lr, eps);
    return GSB_OK;
}

}  // extern "C"
