// featcon.cu -- Eq. 1 feature construction for featureless nodes (SURVEY §8(f)
// f4): F'_v = average of F_u over every in-edge u -> v whose source type has features
// (R-eq1).  One sweep over the full CSC of the featureless type; no sampling.
// Contract: include/gsb.h "Feature construction".
//
// Degrees are power-law, so a warp per node alone leaves a few hub warps (10^4-10^5 in-edges)
// running long after the rest of the grid (MAG240M 1/16 authors: 250 ms per sweep).  Two
// launches instead:
//   head: warp per node; the first kCap edges of each of its relation segments, scaled by
//         1/n (n = all its featured in-edges) and STORED;
//   tail: per relation, the flat edge range of the nodes is cut into pieces of kCap edges and
//         a warp per piece adds (red.add) the scaled sum of the edges in it that lie beyond
//         kCap of their segment.  A node lying wholly inside a piece has <= kCap edges, so only
//         the nodes holding the piece's first and last edge can own such edges: two searches
//         per piece, no list, no workspace.
#include "gsb_internal.cuh"

namespace gsb {

constexpr int64_t kFeatconCap = 128;

// acc[p][.] += rows of edges [e0, e1) of relation r, chunk lane + 32 p of each row.
// keys loaded 32 at a time, 4 source rows in flight per lane per chunk
template <bool BF16, int NP>
__device__ __forceinline__ void featcon_edges(const GraphDev& g, int r, int64_t e0, int64_t e1, int c0, int cpr,
                                              int lane, float (&acc)[NP][Chunk<BF16>::kVec]) {
    const int64_t base = g.node_off[g.src_t[r]];
    for (int64_t cb = e0; cb < e1; cb += 32) {
        const uint4* prow = (cb + lane < e1) ? feat_row(g, base + g.indices[r][cb + lane]) : nullptr;
        const int cnt = (int)min((int64_t)32, e1 - cb);
        for (int k = 0; k < cnt; k += 4) {
            uint4 x[4][NP];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint64_t p = __shfl_sync(0xffffffffu, (uint64_t)prow, (k + u) & 31);
#pragma unroll
                for (int q = 0; q < NP; ++q) {
                    const int c = c0 + lane + 32 * q;
                    x[u][q] = (c < cpr && k + u < cnt) ? __ldg(reinterpret_cast<const uint4*>(p) + c)
                                                       : make_uint4(0u, 0u, 0u, 0u);
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int q = 0; q < NP; ++q) chunk_acc<BF16>(acc[q], x[u][q]);
        }
    }
}

__device__ __forceinline__ int64_t featcon_degree(const GraphDev& g, uint32_t rel_mask, int64_t v) {
    int64_t n = 0;
    for (int r = 0; r < g.R; ++r)
        if ((rel_mask >> r) & 1u) n += g.indptr[r][v + 1] - g.indptr[r][v];
    return n;
}

template <bool BF16, int NP>
__global__ void __launch_bounds__(256) featcon_kernel(GraphDev g, uint32_t rel_mask, int64_t first, int64_t count,
                                                      int dim, float* __restrict__ out) {
    GSB_PDL_ENTRY();
    constexpr int V = Chunk<BF16>::kVec;
    const int lane = threadIdx.x & 31;
    const int cpr = dim / V;                       // 16-byte chunks per row
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < count; i += warps) {
        const int64_t v = first + i;
        const int64_t n = featcon_degree(g, rel_mask, v);
        const float inv = n > 0 ? 1.f / (float)n : 0.f;
        for (int c0 = 0; c0 < cpr; c0 += 32 * NP) {
            float acc[NP][V];
#pragma unroll
            for (int q = 0; q < NP; ++q)
#pragma unroll
                for (int k = 0; k < V; ++k) acc[q][k] = 0.f;
            for (int r = 0; r < g.R; ++r) {
                if (!((rel_mask >> r) & 1u)) continue;
                const int64_t e0 = g.indptr[r][v], e1 = g.indptr[r][v + 1];
                featcon_edges<BF16, NP>(g, r, e0, min(e1, e0 + kFeatconCap), c0, cpr, lane, acc);
            }
#pragma unroll
            for (int q = 0; q < NP; ++q) {
                const int c = c0 + lane + 32 * q;
                if (c >= cpr) continue;
                float4* o = reinterpret_cast<float4*>(out + i * dim + (int64_t)c * V);
#pragma unroll
                for (int k = 0; k < V; k += 4)
                    __stcs(o + k / 4, make_float4(acc[q][k] * inv, acc[q][k + 1] * inv, acc[q][k + 2] * inv,
                                                  acc[q][k + 3] * inv));
            }
        }
    }
}

template <bool BF16, int NP>
__global__ void __launch_bounds__(256) featcon_tail_kernel(GraphDev g, int r, uint32_t rel_mask, int64_t first,
                                                           int64_t count, int dim, float* __restrict__ out) {
    GSB_PDL_ENTRY();
    constexpr int V = Chunk<BF16>::kVec;
    const int lane = threadIdx.x & 31;
    const int cpr = dim / V;
    const int64_t* __restrict__ ip = g.indptr[r];
    const int64_t E0 = ip[first], E1 = ip[first + count];
    const int64_t pieces = (E1 - E0 + kFeatconCap - 1) / kFeatconCap;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t k = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; k < pieces; k += warps) {
        const int64_t a = E0 + k * kFeatconCap, b = min(E1, a + kFeatconCap);
        const int64_t va = seg_find(ip, first, first + count, a, lane);
        const int64_t vb = seg_find(ip, va, first + count, b - 1, lane);
        for (int64_t v = va;; v = vb) {
            const int64_t t0 = max(a, ip[v] + kFeatconCap), t1 = min(b, ip[v + 1]);
            if (t0 < t1) {
                const float inv = 1.f / (float)featcon_degree(g, rel_mask, v);
                for (int c0 = 0; c0 < cpr; c0 += 32 * NP) {
                    float acc[NP][V];
#pragma unroll
                    for (int q = 0; q < NP; ++q)
#pragma unroll
                        for (int j = 0; j < V; ++j) acc[q][j] = 0.f;
                    featcon_edges<BF16, NP>(g, r, t0, t1, c0, cpr, lane, acc);
#pragma unroll
                    for (int q = 0; q < NP; ++q) {
                        const int c = c0 + lane + 32 * q;
                        if (c >= cpr) continue;
                        float* o = out + (v - first) * dim + (int64_t)c * V;
#pragma unroll
                        for (int j = 0; j < V; j += 4)
                            red_add_f4(o + j, make_float4(acc[q][j] * inv, acc[q][j + 1] * inv,
                                                          acc[q][j + 2] * inv, acc[q][j + 3] * inv));
                    }
                }
            }
            if (v == vb) break;
        }
    }
}

template <bool BF16, int NP>
static gsb_status launch_featcon(const GraphDev& g, uint32_t rel_mask, int64_t first, int64_t count, int dim,
                                 float* out, cudaStream_t s) {
    const int grid = grid_for(count * 32, 256, kNumSMs * 8);
    GSB_LAUNCH("featcon", (featcon_kernel<BF16, NP>), grid, 256, 0, s, g, rel_mask, first, count, dim, out);
    for (int r = 0; r < g.R; ++r) {
        if (!((rel_mask >> r) & 1u)) continue;
        GSB_LAUNCH("featcon_tail", (featcon_tail_kernel<BF16, NP>), kNumSMs * 8, 256, 0, s, g, r, rel_mask, first,
                   count, dim, out);
    }
    return GSB_OK;
}

template <bool BF16>
static gsb_status launch_featcon_np(const GraphDev& g, uint32_t rel_mask, int64_t first, int64_t count, int dim,
                                    float* out, cudaStream_t s) {
    const int cpr = dim / Chunk<BF16>::kVec;
    if (cpr <= 32) return launch_featcon<BF16, 1>(g, rel_mask, first, count, dim, out, s);
    if (cpr <= 64) return launch_featcon<BF16, 2>(g, rel_mask, first, count, dim, out, s);
    return launch_featcon<BF16, 3>(g, rel_mask, first, count, dim, out, s);
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
    cudaStream_t s = (cudaStream_t)stream;
    return g.feat_dtype == GSB_BF16 ? launch_featcon_np<true>(g, rel_mask, first, count, dim, out, s)
                                    : launch_featcon_np<false>(g, rel_mask, first, count, dim, out, s);
}
