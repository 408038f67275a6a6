// featcon.cu -- Eq. 1 feature construction for featureless nodes (SURVEY §8(f)
// f4): F'_v = average of F_u over every in-edge u -> v whose source type has features
// (R-eq1).  One sweep over the full CSC of the featureless type; no sampling.
// Contract: include/gsb.h "Feature construction".
#include "gsb_internal.cuh"

namespace gsb {

// warp per dst node; lanes over 16-byte chunks of the source rows (several passes for rows
// wider than 512 B); 4 source rows in flight per lane, keys loaded 32 at a time.
template <bool BF16>
__global__ void __launch_bounds__(256) featcon_kernel(GraphDev g, int ntype, uint32_t rel_mask, int64_t first,
                                                      int64_t count, int dim, float* __restrict__ out) {
    GSB_PDL_ENTRY();
    constexpr int V = Chunk<BF16>::kVec;
    const int lane = threadIdx.x & 31;
    const int cpr = dim / V;                       // 16-byte chunks per row
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < count; i += warps) {
        const int64_t v = first + i;
        for (int c0 = 0; c0 < cpr; c0 += 32) {
            const int c = c0 + lane;
            const bool cl = c < cpr;
            float acc[V];
#pragma unroll
            for (int k = 0; k < V; ++k) acc[k] = 0.f;
            int64_t n = 0;
            for (int r = 0; r < g.R; ++r) {
                if (!((rel_mask >> r) & 1u)) continue;
                const int64_t e0 = g.indptr[r][v], e1 = g.indptr[r][v + 1];
                n += e1 - e0;
                const int64_t base = g.node_off[g.src_t[r]];
                for (int64_t cb = e0; cb < e1; cb += 32) {
                    const int64_t key = (cb + lane < e1) ? base + g.indices[r][cb + lane] : 0;
                    const uint4* prow = (cb + lane < e1) ? feat_row(g, key) : nullptr;
                    const int cnt = (int)min((int64_t)32, e1 - cb);
                    for (int k = 0; k < cnt; k += 4) {
                        uint4 x[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const uint64_t p = __shfl_sync(0xffffffffu, (uint64_t)prow, (k + u) & 31);
                            x[u] = (cl && k + u < cnt) ? __ldg(reinterpret_cast<const uint4*>(p) + c)
                                                       : make_uint4(0u, 0u, 0u, 0u);
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u) chunk_acc<BF16>(acc, x[u]);
                    }
                }
            }
            if (cl) {
                const float inv = n > 0 ? 1.f / (float)n : 0.f;
                float* o = out + i * dim + (int64_t)c * V;
#pragma unroll
                for (int k = 0; k < V; k += 4)
                    *reinterpret_cast<float4*>(o + k) = make_float4(acc[k] * inv, acc[k + 1] * inv, acc[k + 2] * inv,
                                                                    acc[k + 3] * inv);
            }
        }
    }
}

}  // namespace gsb

using namespace gsb;

extern "C" gsb_status gsb_construct_features(gsb_graph_t gh, int32_t ntype, uint32_t featured_mask, int64_t first,
                                             int64_t count, float* out, int32_t dim, void* stream) {
    Graph* G = reinterpret_cast<Graph*>(gh);
    GSB_CHECK_ARG(G && out && ntype >= 0 && ntype < G->dev.T, "bad argument");
    GSB_CHECK_ARG(first >= 0 && count >= 0 && first + count <= G->counts[ntype], "rows [%lld, %lld) outside ntype %d",
                  (long long)first, (long long)(first + count), ntype);
    const GraphDev& g = G->dev;
    uint32_t rel_mask = 0;
    for (int r = 0; r < g.R; ++r) {
        if (g.dst_t[r] != ntype || !((featured_mask >> g.src_t[r]) & 1u)) continue;
        const int t = g.src_t[r];
        GSB_CHECK_ARG(g.indptr[r] && g.indices[r], "CSC of etype %d not built", r);
        GSB_CHECK_ARG(g.feat[t] || g.nparts > 1, "features of ntype %d not registered", t);
        GSB_CHECK_ARG(g.dim_t[t] == dim, "featured ntype %d has width %d, expected %d", t, g.dim_t[t], dim);
        rel_mask |= 1u << r;
    }
    const int vec = g.feat_dtype == GSB_BF16 ? 8 : 4;
    GSB_CHECK_ARG(dim > 0 && dim % vec == 0, "dim %d must be a multiple of %d", dim, vec);
    if (count == 0) return GSB_OK;
    const int grid = grid_for(count * 32, 256, kNumSMs * 8);
    cudaStream_t s = (cudaStream_t)stream;
    if (g.feat_dtype == GSB_BF16)
        GSB_LAUNCH("featcon", featcon_kernel<true>, grid, 256, 0, s, g, ntype, rel_mask, first, count, dim, out);
    else
        GSB_LAUNCH("featcon", featcon_kernel<false>, grid, 256, 0, s, g, ntype, rel_mask, first, count, dim, out);
    return GSB_OK;
}
