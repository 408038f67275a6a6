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

}  // extern "C"
