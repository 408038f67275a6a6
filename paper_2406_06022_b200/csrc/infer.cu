// infer.cu -- full-graph layer-wise inference support:
// the block's input rows as int32 row ids into an all-node embedding table (layer l >= 1
// reads h_{l-1} of every node through this map), and NC accuracy of the decoder.
// Contract: include/gsb.h "Full-graph inference".
#include "gsb_internal.cuh"

namespace gsb {

__global__ void input_rowmap_kernel(const HopMeta* __restrict__ m, const int64_t* __restrict__ src_gid, int64_t base,
                                    int32_t* __restrict__ rowmap) {
    GSB_PDL_ENTRY();
    const int64_t n = m->n_src;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        rowmap[i] = (int32_t)(src_gid[i] - base);
}

// warp per row: logits row (already h Wc) + bc, argmax (lowest class on ties), compare
__global__ void __launch_bounds__(256) nc_argmax_kernel(const float* __restrict__ logits, int64_t ldl, int64_t n,
                                                        int C, const float* __restrict__ bc,
                                                        const int32_t* __restrict__ labels,
                                                        const int64_t* __restrict__ seed_gid, int64_t base,
                                                        int32_t* __restrict__ pred,
                                                        unsigned long long* __restrict__ correct) {
    GSB_PDL_ENTRY();
    const int lane = threadIdx.x & 31;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
        float best = -INFINITY;
        int arg = 0x7fffffff;
        for (int c = lane; c < C; c += 32) {
            const float x = logits[i * ldl + c] + bc[c];
            if (x > best) { best = x; arg = c; }
        }
        for (int o = 16; o; o >>= 1) {
            const float ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int oa = __shfl_xor_sync(0xffffffffu, arg, o);
            if (ob > best || (ob == best && oa < arg)) { best = ob; arg = oa; }
        }
        if (lane == 0) {
            if (pred) pred[i] = arg;
            if (correct && arg == labels[seed_gid[i] - base]) atomicAdd(correct, 1ull);
        }
    }
}

}  // namespace gsb

using namespace gsb;

extern "C" {

gsb_status gsb_blocks_input_rowmap(gsb_blocks_t b, const void* arena, int64_t gid_base, int32_t* rowmap,
                                   void* stream) {
    Blocks* B = reinterpret_cast<Blocks*>(b);
    GSB_CHECK_ARG(B && arena && rowmap, "null argument");
    GSB_CHECK_ARG(B->g->total_nodes - gid_base <= INT32_MAX, "row ids exceed int32");
    HopBufs hb = B->hop(B->L, const_cast<void*>(arena));
    GSB_LAUNCH("input_rowmap", input_rowmap_kernel, grid_for(hb.cap_src, 256, kNumSMs * 8), 256, 0,
               (cudaStream_t)stream, hb.meta, hb.src_gid, gid_base, rowmap);
    return GSB_OK;
}

gsb_status gsb_nc_predict(const float* h, int64_t n, int32_t d, const float* Wc, const float* bc, int32_t C,
                          const int32_t* labels, const int64_t* seed_gid, int64_t label_gid_base, float* logits_ws,
                          int32_t* pred, unsigned long long* correct, void* stream) {
    GSB_CHECK_ARG(h && Wc && bc && logits_ws && n >= 0 && d > 0 && d % 32 == 0 && C >= 1, "bad argument");
    GSB_CHECK_ARG(!correct || (labels && seed_gid), "accuracy needs labels and seed gids");
    if (n == 0) return GSB_OK;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t ldl = (C + 3) / 4 * 4;
    gsb_status st = gsb_gemm(0, h, d, Wc, C, n, C, d, logits_ws, ldl, s);     // logits = h Wc (tcgen05)
    if (st != GSB_OK) return st;
    GSB_LAUNCH("nc_argmax", nc_argmax_kernel, grid_for(n * 32, 256, kNumSMs * 8), 256, 0, s, logits_ws, ldl, n, C, bc,
               labels, seed_gid, label_gid_base, pred, correct);
    return GSB_OK;
}

}  // extern "C"
