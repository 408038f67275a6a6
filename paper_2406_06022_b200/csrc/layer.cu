// layer.cu -- RGCN layer forward / backward and the NC decoder + softmax-CE loss.
// Contract: include/gsb.h "RGCN layer" and "Node-classification decoder".
#include "gemm_tma3.cuh"
#include "gsb_internal.cuh"

namespace gsb {

// ------------------------------------------------------------------------------------
// aggregation: warp per dst row j
//   Acat[j, s*d + :] = mean_{e in seg(j,s)} h_src[e_src[e], :]    (0 when empty)
//   Acat[j, S_t*d + :] = h_src[self(j), :]
// Source rows are read in 16-byte chunks (4 fp32 or 8 bf16 values, widened exactly to
// fp32); LPE lanes cover one row's chunks and the warp's 32/LPE lane groups take
// different edges of the segment (4 rows in flight per lane), reduced by shuffles at the
// end -- so narrow rows (64-d fp32, 128-d bf16) still keep every lane loading.
// ------------------------------------------------------------------------------------
template <bool FEAT>
__device__ __forceinline__ const uint4* src_row(const GraphDev& g, const char* h, int row_bytes, int64_t key,
                                                const int32_t* rowmap) {
    if (FEAT) return feat_row(g, key);              // layer 0: fused gather by gid (a5)
    const int64_t row = rowmap ? (int64_t)rowmap[key] : key;   // exchange order (partitioned features)
    return reinterpret_cast<const uint4*>(h + row * row_bytes);
}

// FEAT: source rows come from the feature tables via e_src_gid / dst_gid (no x0 buffer)
template <bool FEAT, bool BF16, int LPE>
#ifndef GSB_AGG_MINB
#define GSB_AGG_MINB 5
#endif
#ifndef GSB_AGG_BPS
#define GSB_AGG_BPS 5
#endif
__global__ void __launch_bounds__(256, GSB_AGG_MINB) agg_kernel(GraphDev g, const HopMeta* __restrict__ m,
                                                  const int64_t* __restrict__ seg_ptr,
                                                  const int32_t* __restrict__ e_src,
                                                  const int64_t* __restrict__ e_src_gid,
                                                  const int64_t* __restrict__ dst_gid, const char* __restrict__ h,
                                                  int row_bytes, int d, float* __restrict__ acat, int64_t lda,
                                                  const int32_t* __restrict__ rowmap, int64_t seg_cap) {
    GSB_PDL_ENTRY();
    constexpr int V = Chunk<BF16>::kVec;
    constexpr int G = 32 / LPE;                  // edges per warp pass
    __shared__ int64_t s_dst_off[kMaxT + 1], s_src_off[kMaxT + 1];
    if (threadIdx.x <= (unsigned)g.T) {
        s_dst_off[threadIdx.x] = m->dst_off[threadIdx.x];
        s_src_off[threadIdx.x] = m->src_off[threadIdx.x];
    }
    const int64_t n = m->n_dst;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int grp = lane / LPE, sub = lane % LPE;
    const int S = g.S;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int cpr = row_bytes >> 4;              // 16-byte chunks per row
    for (int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; j < n; j += warps) {
        int t = 0;
        for (int k = 1; k < g.T; ++k) t += (j >= s_dst_off[k]) ? 1 : 0;
        const int St = g.n_slots[t];
        float* out = acat + j * lda;
        // all St+1 slot boundaries of row j with one load (lane s = start of slot s)
        const int64_t bl = (lane <= St) ? seg_ptr[j * S + lane] : 0;
        // the self row's address, resolved while the segments load
        const uint4* ps = src_row<FEAT>(g, h, row_bytes, FEAT ? dst_gid[j] : s_src_off[t] + (j - s_dst_off[t]), rowmap);
        for (int s = 0; s < St; ++s) {
            const int64_t e0 = __shfl_sync(0xffffffffu, bl, s), e1 = __shfl_sync(0xffffffffu, bl, s + 1);
            const float inv = (e1 > e0) ? 1.f / (float)(e1 - e0) : 0.f;
            // every lane runs every chunk pass (the shuffles need the whole warp); lanes past
            // the row width or the segment end only predicate their loads and stores
            for (int c0 = 0; c0 < cpr; c0 += LPE) {
                const int c = c0 + sub;
                const bool cl = c < cpr;
                float acc[V];
#pragma unroll
                for (int v = 0; v < V; ++v) acc[v] = 0.f;
                // a segment longer than seg_cap (fanout ALL hubs) leaves its tail to heavy_kernel
                const int64_t ec = (e1 - e0 > seg_cap) ? e0 + seg_cap : e1;
                for (int64_t cb = e0; cb < ec; cb += 32) {
                    // one coalesced load of up to 32 source keys; lane i resolves the row
                    // address of edge cb+i once, the warp takes the addresses by shuffle
                    const uint4* prow = (cb + lane < ec)
                        ? src_row<FEAT>(g, h, row_bytes, FEAT ? e_src_gid[cb + lane] : (int64_t)e_src[cb + lane], rowmap)
                        : nullptr;
                    const int cnt = (int)min((int64_t)32, ec - cb);
                    for (int k = 0; k < cnt; k += 4 * G) {
                        uint4 x[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int idx = k + grp + G * u;
                            const uint64_t pu = __shfl_sync(0xffffffffu, (uint64_t)prow, idx & 31);
                            x[u] = make_uint4(0u, 0u, 0u, 0u);
                            if (cl && idx < cnt) x[u] = __ldg(reinterpret_cast<const uint4*>(pu) + c);
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u) chunk_acc<BF16>(acc, x[u]);
                    }
                }
#pragma unroll
                for (int o = LPE; o < 32; o <<= 1)
#pragma unroll
                    for (int v = 0; v < V; ++v) acc[v] += __shfl_xor_sync(0xffffffffu, acc[v], o);
                if (cl && grp == 0) {
                    float4* o4 = reinterpret_cast<float4*>(out + (int64_t)s * d + (int64_t)c * V);
#pragma unroll
                    for (int v = 0; v < V; v += 4)
                        o4[v / 4] = make_float4(acc[v] * inv, acc[v + 1] * inv, acc[v + 2] * inv, acc[v + 3] * inv);
                }
            }
        }
        for (int c = lane; c < cpr; c += 32) {
            float r[V];
#pragma unroll
            for (int v = 0; v < V; ++v) r[v] = 0.f;
            chunk_acc<BF16>(r, __ldg(ps + c));
            float4* o4 = reinterpret_cast<float4*>(out + (int64_t)St * d + (int64_t)c * V);
#pragma unroll
            for (int v = 0; v < V; v += 4) o4[v / 4] = make_float4(r[v], r[v + 1], r[v + 2], r[v + 3]);
        }
    }
}

// ------------------------------------------------------------------------------------
// aggregation, half-warp per dst row (layer 0, rows of >= 256 B): the two 16-lane halves of a
// warp run two dst rows side by side, so the dependent chain of each segment (key load ->
// row address -> row loads) of one row overlaps the other's; 16 lanes x 16 B cover 256 B of
// a source row per pass, 4 source rows in flight per lane, no cross-lane reduction.  The
// halves diverge freely (own loop trip counts); every shuffle names only its half.
// Requires S < 16 (a row's slot boundaries live in one lane each of its half).  Taken for
// 256-B rows of large batches (launch_agg_lpe).
// ------------------------------------------------------------------------------------
#ifndef GSB_AGG_HALF
#define GSB_AGG_HALF 1
#endif
template <bool FEAT, bool BF16>
__global__ void __launch_bounds__(256, GSB_AGG_MINB) agg_half_kernel(
    GraphDev g, const HopMeta* __restrict__ m, const int64_t* __restrict__ seg_ptr, const int32_t* __restrict__ e_src,
    const int64_t* __restrict__ e_src_gid, const int64_t* __restrict__ dst_gid, const char* __restrict__ h,
    int row_bytes, int d, float* __restrict__ acat, int64_t lda, const int32_t* __restrict__ rowmap, int64_t seg_cap) {
    GSB_PDL_ENTRY();
    constexpr int V = Chunk<BF16>::kVec;
    __shared__ int64_t s_dst_off[kMaxT + 1], s_src_off[kMaxT + 1];
    if (threadIdx.x <= (unsigned)g.T) {
        s_dst_off[threadIdx.x] = m->dst_off[threadIdx.x];
        s_src_off[threadIdx.x] = m->src_off[threadIdx.x];
    }
    const int64_t n = m->n_dst;
    __syncthreads();
    const int lane = threadIdx.x & 31, hl = lane & 15;
    const unsigned hmask = (lane < 16) ? 0x0000ffffu : 0xffff0000u;
    const int S = g.S;
    const int64_t halves = ((int64_t)gridDim.x * blockDim.x) >> 4;
    const int cpr = row_bytes >> 4;
    for (int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 4; j < n; j += halves) {
        int t = 0;
        for (int k = 1; k < g.T; ++k) t += (j >= s_dst_off[k]) ? 1 : 0;
        const int St = g.n_slots[t];
        float* out = acat + j * lda;
        const int64_t bl = (hl <= St) ? seg_ptr[j * S + hl] : 0;
        const uint4* ps = src_row<FEAT>(g, h, row_bytes, FEAT ? dst_gid[j] : s_src_off[t] + (j - s_dst_off[t]), rowmap);
        for (int s = 0; s < St; ++s) {
            const int64_t e0 = __shfl_sync(hmask, bl, s, 16), e1 = __shfl_sync(hmask, bl, s + 1, 16);
            const float inv = (e1 > e0) ? 1.f / (float)(e1 - e0) : 0.f;
            const int64_t ec = (e1 - e0 > seg_cap) ? e0 + seg_cap : e1;
            for (int c0 = 0; c0 < cpr; c0 += 16) {
                const int c = c0 + hl;
                const bool cl = c < cpr;
                float acc[V];
#pragma unroll
                for (int v = 0; v < V; ++v) acc[v] = 0.f;
                for (int64_t cb = e0; cb < ec; cb += 16) {
                    const uint4* prow = (cb + hl < ec)
                        ? src_row<FEAT>(g, h, row_bytes, FEAT ? e_src_gid[cb + hl] : (int64_t)e_src[cb + hl], rowmap)
                        : nullptr;
                    const int cnt = (int)min((int64_t)16, ec - cb);
                    for (int k = 0; k < cnt; k += 4) {
                        uint4 x[4];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const uint64_t pu = __shfl_sync(hmask, (uint64_t)prow, (k + u) & 15, 16);
                            x[u] = make_uint4(0u, 0u, 0u, 0u);
                            if (cl && k + u < cnt) x[u] = __ldg(reinterpret_cast<const uint4*>(pu) + c);
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u) chunk_acc<BF16>(acc, x[u]);
                    }
                }
                if (cl) {
                    float4* o4 = reinterpret_cast<float4*>(out + (int64_t)s * d + (int64_t)c * V);
#pragma unroll
                    for (int v = 0; v < V; v += 4)
                        o4[v / 4] = make_float4(acc[v] * inv, acc[v + 1] * inv, acc[v + 2] * inv, acc[v + 3] * inv);
                }
            }
        }
        for (int c = hl; c < cpr; c += 16) {
            float r[V];
#pragma unroll
            for (int v = 0; v < V; ++v) r[v] = 0.f;
            chunk_acc<BF16>(r, __ldg(ps + c));
            float4* o4 = reinterpret_cast<float4*>(out + (int64_t)St * d + (int64_t)c * V);
#pragma unroll
            for (int v = 0; v < V; v += 4) o4[v / 4] = make_float4(r[v], r[v + 1], r[v + 2], r[v + 3]);
        }
    }
}

// ------------------------------------------------------------------------------------
// aggregation, segment-parallel (default): a group of LPE lanes owns one (dst row j, slot s)
// unit -- a relation's segment (its mean) or the self slot (the dst's own row) -- and each
// lane owns 32 bytes of the row (LPE = row bytes / 32: 8 lanes for 128-d bf16 or 64-d fp32,
// 16 for 128-d fp32).  Every lane walks the segment's edges itself, U source rows in flight
// (256-bit loads, LDG.E.ENL2.256), and sums in registers: no cross-lane reduction, no
// shuffles, and empty slots cost one store.  A warp's 32/LPE groups take consecutive units.
// ------------------------------------------------------------------------------------
template <bool W256 = true>
__device__ __forceinline__ void ldg256(const void* p, uint32_t (&r)[8]) {
    if (!W256) {
        const uint4 a = __ldg(reinterpret_cast<const uint4*>(p)), b = __ldg(reinterpret_cast<const uint4*>(p) + 1);
        r[0] = a.x; r[1] = a.y; r[2] = a.z; r[3] = a.w; r[4] = b.x; r[5] = b.y; r[6] = b.z; r[7] = b.w;
        return;
    }
    asm volatile("ld.global.nc.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "l"(p));
}
template <bool BF16>
__device__ __forceinline__ void acc256(float* acc, const uint32_t (&r)[8]) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        if (BF16) {
            acc[2 * i] += bf16_lo(r[i]);
            acc[2 * i + 1] += bf16_hi(r[i]);
        } else {
            acc[i] += __uint_as_float(r[i]);
        }
    }
}

template <bool FEAT, bool BF16, int LPE, int U, bool W256 = true>
__global__ void __launch_bounds__(256) agg_seg_kernel(GraphDev g, const HopMeta* __restrict__ m,
                                                      const int64_t* __restrict__ seg_ptr,
                                                      const int32_t* __restrict__ e_src,
                                                      const int64_t* __restrict__ e_src_gid,
                                                      const int64_t* __restrict__ dst_gid, const char* __restrict__ h,
                                                      int row_bytes, int d, float* __restrict__ acat, int64_t lda,
                                                      const int32_t* __restrict__ rowmap, int64_t seg_cap) {
    GSB_PDL_ENTRY();
    constexpr int V = BF16 ? 16 : 8;            // floats per lane (32 bytes of the row)
    __shared__ int64_t s_dst_off[kMaxT + 1], s_src_off[kMaxT + 1];
    if (threadIdx.x <= (unsigned)g.T) {
        s_dst_off[threadIdx.x] = m->dst_off[threadIdx.x];
        s_src_off[threadIdx.x] = m->src_off[threadIdx.x];
    }
    const int64_t n = m->n_dst;
    __syncthreads();
    const int sub = threadIdx.x % LPE;
    const int S = g.S;
    const uint32_t S1 = (uint32_t)S + 1;
    const uint32_t units = (uint32_t)(n * S1);
    const uint32_t groups = gridDim.x * (blockDim.x / LPE);
    for (uint32_t u = blockIdx.x * (blockDim.x / LPE) + threadIdx.x / LPE; u < units; u += groups) {
        const uint32_t j = u / S1;
        const int s = (int)(u - j * S1);
        int t = 0;
        for (int k = 1; k < g.T; ++k) t += ((int64_t)j >= s_dst_off[k]) ? 1 : 0;
        const int St = g.n_slots[t];
        if (s > St) continue;
        float acc[V];
#pragma unroll
        for (int v = 0; v < V; ++v) acc[v] = 0.f;
        if (s == St) {          // self slot: the dst's own row
            const char* row = FEAT ? reinterpret_cast<const char*>(feat_row(g, dst_gid[j]))
                                   : reinterpret_cast<const char*>(
                                         src_row<false>(g, h, row_bytes, s_src_off[t] + ((int64_t)j - s_dst_off[t]), rowmap));
            uint32_t r[8];
            ldg256<W256>(row + sub * 32, r);
            acc256<BF16>(acc, r);
        } else {
            const int64_t e0 = seg_ptr[(int64_t)j * S + s], e1 = seg_ptr[(int64_t)j * S + s + 1];
            // a segment longer than seg_cap (fanout ALL hubs) leaves its tail to heavy_kernel
            const int64_t ec = (e1 - e0 > seg_cap) ? e0 + seg_cap : e1;
            for (int64_t e = e0; e < ec; e += U) {
                const char* p[U];
#pragma unroll
                for (int k = 0; k < U; ++k)
                    p[k] = (e + k < ec) ? reinterpret_cast<const char*>(src_row<FEAT>(
                                              g, h, row_bytes, FEAT ? e_src_gid[e + k] : (int64_t)e_src[e + k], rowmap))
                                        : nullptr;
                uint32_t r[U][8];
#pragma unroll
                for (int k = 0; k < U; ++k) {
                    if (p[k]) {
                        ldg256<W256>(p[k] + sub * 32, r[k]);
                    } else {
#pragma unroll
                        for (int i = 0; i < 8; ++i) r[k][i] = 0u;
                    }
                }
#pragma unroll
                for (int k = 0; k < U; ++k) acc256<BF16>(acc, r[k]);
            }
            const float inv = (e1 > e0) ? 1.f / (float)(e1 - e0) : 0.f;
#pragma unroll
            for (int v = 0; v < V; ++v) acc[v] *= inv;
        }
        float4* o4 = reinterpret_cast<float4*>(acat + (int64_t)j * lda + (int64_t)s * d + (int64_t)sub * V);
#pragma unroll
        for (int v = 0; v < V; v += 4) o4[v / 4] = make_float4(acc[v], acc[v + 1], acc[v + 2], acc[v + 3]);
    }
}

template <bool FEAT, bool BF16>
static gsb_status launch_agg_seg(const char* name, cudaStream_t s, const GraphDev& g, const HopBufs& hb, const char* h,
                                 int row_bytes, int d, float* acat, int64_t lda, const int32_t* rowmap,
                                 int64_t seg_cap) {
    const int lpe = row_bytes / 32;
    const int64_t units = hb.cap_dst * (g.S + 1);
    // one wave of resident blocks (A/B knobs: GSB_AGG_BPS blocks per SM, GSB_AGG_U rows in flight)
    static const int bps = getenv("GSB_AGG_BPS") ? atoi(getenv("GSB_AGG_BPS")) : 4;
    static const int uu = getenv("GSB_AGG_U") ? atoi(getenv("GSB_AGG_U")) : 8;
    const int grid = grid_for(units * lpe, 256, kNumSMs * bps);
#define GSB_AGG_SEG(L, UU)                                                                                       \
    GSB_LAUNCH(name, (agg_seg_kernel<FEAT, BF16, L, UU>), grid, 256, 0, s, g, hb.meta, hb.seg_ptr, hb.e_src,     \
               hb.e_src_gid, hb.dst_gid, h, row_bytes, d, acat, lda, rowmap, seg_cap)
    static const bool w128 = getenv("GSB_AGG_W") && atoi(getenv("GSB_AGG_W")) == 128;
    if (w128 && lpe == 8 && uu == 8) {
        GSB_LAUNCH(name, (agg_seg_kernel<FEAT, BF16, 8, 8, false>), grid, 256, 0, s, g, hb.meta, hb.seg_ptr, hb.e_src,
                   hb.e_src_gid, hb.dst_gid, h, row_bytes, d, acat, lda, rowmap, seg_cap);
    } else if (uu == 4) {
        if (lpe == 4) GSB_AGG_SEG(4, 4);
        else if (lpe == 8) GSB_AGG_SEG(8, 4);
        else if (lpe == 16) GSB_AGG_SEG(16, 4);
        else GSB_AGG_SEG(32, 4);
    } else {
        if (lpe == 4) GSB_AGG_SEG(4, 8);
        else if (lpe == 8) GSB_AGG_SEG(8, 8);
        else if (lpe == 16) GSB_AGG_SEG(16, 8);
        else GSB_AGG_SEG(32, 8);
    }
#undef GSB_AGG_SEG
    return GSB_OK;
}

// quarter-warp per dst row (256-B rows): 8 lanes x 32 B (256-bit loads) cover a source row,
// four dst rows per warp side by side -- four dependent segment chains in flight per warp
// (mag: ~3 rows per warp of the warp kernel's grid).  Default for 256-B feature rows with
// S < 8: mag layer 0 34.2 us (0.417 of HBM) vs 35.2 for the warp kernel, step 0.2009-0.2012 vs
// 0.2036-0.2040 ms (profiles/round2_agg_ab.md).
#ifndef GSB_AGG_QMINB
#define GSB_AGG_QMINB 4       // 64 registers (3: 76-80, slower kernel: 38.5 vs 34.2 us on mag)
#endif
template <bool FEAT, bool BF16>
__global__ void __launch_bounds__(256, GSB_AGG_QMINB) agg_quarter_kernel(
    GraphDev g, const HopMeta* __restrict__ m, const int64_t* __restrict__ seg_ptr, const int32_t* __restrict__ e_src,
    const int64_t* __restrict__ e_src_gid, const int64_t* __restrict__ dst_gid, const char* __restrict__ h,
    int row_bytes, int d, float* __restrict__ acat, int64_t lda, const int32_t* __restrict__ rowmap, int64_t seg_cap) {
    GSB_PDL_ENTRY();
    constexpr int L = 8;
    constexpr int V = 2 * Chunk<BF16>::kVec;      // values per lane (32 B)
    __shared__ int64_t s_dst_off[kMaxT + 1], s_src_off[kMaxT + 1];
    if (threadIdx.x <= (unsigned)g.T) {
        s_dst_off[threadIdx.x] = m->dst_off[threadIdx.x];
        s_src_off[threadIdx.x] = m->src_off[threadIdx.x];
    }
    const int64_t n = m->n_dst;
    __syncthreads();
    const int lane = threadIdx.x & 31, ql = lane & (L - 1);
    const unsigned qmask = 0xffu << (lane & ~(L - 1));
    const int S = g.S;
    const int64_t quarters = ((int64_t)gridDim.x * blockDim.x) / L;
    for (int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / L; j < n; j += quarters) {
        int t = 0;
        for (int k = 1; k < g.T; ++k) t += (j >= s_dst_off[k]) ? 1 : 0;
        const int St = g.n_slots[t];
        float* out = acat + j * lda;
        const int64_t bl = (ql <= St) ? seg_ptr[j * S + ql] : 0;
        const char* ps = reinterpret_cast<const char*>(
            src_row<FEAT>(g, h, row_bytes, FEAT ? dst_gid[j] : s_src_off[t] + (j - s_dst_off[t]), rowmap));
        for (int s = 0; s < St; ++s) {
            const int64_t e0 = __shfl_sync(qmask, bl, s, L), e1 = __shfl_sync(qmask, bl, s + 1, L);
            const float inv = (e1 > e0) ? 1.f / (float)(e1 - e0) : 0.f;
            const int64_t ec = (e1 - e0 > seg_cap) ? e0 + seg_cap : e1;
            float acc[V];
#pragma unroll
            for (int v = 0; v < V; ++v) acc[v] = 0.f;
            for (int64_t cb = e0; cb < ec; cb += L) {
                const char* prow = (cb + ql < ec)
                    ? reinterpret_cast<const char*>(src_row<FEAT>(g, h, row_bytes,
                                                                  FEAT ? e_src_gid[cb + ql] : (int64_t)e_src[cb + ql], rowmap))
                    : nullptr;
                const int cnt = (int)min((int64_t)L, ec - cb);
                for (int k = 0; k < cnt; k += 4) {
                    uint32_t x[4][8];
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        const uint64_t pu = __shfl_sync(qmask, (uint64_t)prow, (k + u) & (L - 1), L);
#pragma unroll
                        for (int w = 0; w < 8; ++w) x[u][w] = 0u;
                        if (k + u < cnt) ldg256(reinterpret_cast<const char*>(pu) + 32 * ql, x[u]);
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        chunk_acc<BF16>(acc, make_uint4(x[u][0], x[u][1], x[u][2], x[u][3]));
                        chunk_acc<BF16>(acc + V / 2, make_uint4(x[u][4], x[u][5], x[u][6], x[u][7]));
                    }
                }
            }
            float4* o4 = reinterpret_cast<float4*>(out + (int64_t)s * d + (int64_t)ql * V);
#pragma unroll
            for (int v = 0; v < V; v += 4)
                o4[v / 4] = make_float4(acc[v] * inv, acc[v + 1] * inv, acc[v + 2] * inv, acc[v + 3] * inv);
        }
        {
            uint32_t x[8];
            ldg256(ps + 32 * ql, x);
            float r[V];
#pragma unroll
            for (int v = 0; v < V; ++v) r[v] = 0.f;
            chunk_acc<BF16>(r, make_uint4(x[0], x[1], x[2], x[3]));
            chunk_acc<BF16>(r + V / 2, make_uint4(x[4], x[5], x[6], x[7]));
            float4* o4 = reinterpret_cast<float4*>(out + (int64_t)St * d + (int64_t)ql * V);
#pragma unroll
            for (int v = 0; v < V; v += 4) o4[v / 4] = make_float4(r[v], r[v + 1], r[v + 2], r[v + 3]);
        }
    }
}

template <bool FEAT, bool BF16>
static gsb_status launch_agg_lpe(const char* name, int grid, cudaStream_t s, const GraphDev& g, const HopBufs& hb,
                                 const char* h, int row_bytes, int d, float* acat, int64_t lda, const int32_t* rowmap,
                                 int64_t seg_cap) {
    const int cpr = row_bytes / 16;
    // GSB_AGG_HALF (A/B, tests): unset = the choice below, 0 = warp kernel, 2 = half-warp kernel
    // whenever it applies, 4 = quarter-warp kernel whenever it applies.  256-B feature rows with
    // S < 8 take the quarter-warp kernel; else 256-B rows of large batches the half-warp kernel
    // (amazon_lp 290 -> 223 us; the seed capacity is the host-side proxy for the row count);
    // 512-B rows (two passes per segment in the narrower kernels: 45.5 vs 55.8 us) and the rest
    // the warp kernel (profiles/round2_agg_ab.md).
    const char* hk = getenv("GSB_AGG_HALF");
    const bool half_off = hk && strcmp(hk, "0") == 0, half_force = hk && strcmp(hk, "2") == 0;
    const bool many_rows = hb.cap_seeds >= 4 * (int64_t)kNumSMs * 8;
    const bool quarter = !hk || strcmp(hk, "4") == 0;     // default (GSB_AGG_HALF=0 / 2 select the others)
    if (quarter && FEAT && cpr == 16 && g.S < 8 && (reinterpret_cast<uintptr_t>(acat) & 15) == 0 && (lda & 3) == 0) {
        GSB_LAUNCH(name, (agg_quarter_kernel<FEAT, BF16>), kNumSMs * GSB_AGG_QMINB, 256, 0, s, g, hb.meta, hb.seg_ptr,
                   hb.e_src, hb.e_src_gid, hb.dst_gid, h, row_bytes, d, acat, lda, rowmap, seg_cap);
        return GSB_OK;
    }
    if (GSB_AGG_HALF && !half_off && FEAT && cpr == 16 && g.S < 16 && (many_rows || half_force)) {
        GSB_LAUNCH(name, (agg_half_kernel<FEAT, BF16>), grid, 256, 0, s, g, hb.meta, hb.seg_ptr, hb.e_src, hb.e_src_gid,
                   hb.dst_gid, h, row_bytes, d, acat, lda, rowmap, seg_cap);
        return GSB_OK;
    }
    if (cpr <= 4) {
        GSB_LAUNCH(name, (agg_kernel<FEAT, BF16, 4>), grid, 256, 0, s, g, hb.meta, hb.seg_ptr, hb.e_src, hb.e_src_gid,
                   hb.dst_gid, h, row_bytes, d, acat, lda, rowmap, seg_cap);
    } else if (cpr <= 8) {
        GSB_LAUNCH(name, (agg_kernel<FEAT, BF16, 8>), grid, 256, 0, s, g, hb.meta, hb.seg_ptr, hb.e_src, hb.e_src_gid,
                   hb.dst_gid, h, row_bytes, d, acat, lda, rowmap, seg_cap);
    } else if (cpr <= 16) {
        GSB_LAUNCH(name, (agg_kernel<FEAT, BF16, 16>), grid, 256, 0, s, g, hb.meta, hb.seg_ptr, hb.e_src, hb.e_src_gid,
                   hb.dst_gid, h, row_bytes, d, acat, lda, rowmap, seg_cap);
    } else {
        GSB_LAUNCH(name, (agg_kernel<FEAT, BF16, 32>), grid, 256, 0, s, g, hb.meta, hb.seg_ptr, hb.e_src, hb.e_src_gid,
                   hb.dst_gid, h, row_bytes, d, acat, lda, rowmap, seg_cap);
    }
    return GSB_OK;
}

// ------------------------------------------------------------------------------------
// Heavy segments (fanout ALL, e.g. full-graph inference over hub nodes): agg_kernel sums the
// first kSegCap edges of every segment.  The hop's flat edge range is cut into pieces of
// kSegCap edges; a warp per piece adds the scaled sum of the edges in it that lie beyond
// kSegCap of their (row, slot) segment into the Acat slot row (red.add; agg_kernel's store of
// the head precedes it in stream order).  A segment wholly inside a piece has <= kSegCap
// edges, so only the segments holding the piece's first and last edge qualify: a hub's tail
// is spread over (len - kSegCap) / kSegCap warps, with no list and no workspace.
// ------------------------------------------------------------------------------------
constexpr int64_t kSegCap = 256;

template <bool FEAT, bool BF16, int LPE>
__global__ void __launch_bounds__(256) heavy_kernel(GraphDev g, const HopMeta* __restrict__ m,
                                                    const int64_t* __restrict__ seg_ptr,
                                                    const int32_t* __restrict__ e_src,
                                                    const int64_t* __restrict__ e_src_gid, const char* __restrict__ h,
                                                    int row_bytes, int d, float* __restrict__ acat, int64_t lda,
                                                    const int32_t* __restrict__ rowmap) {
    GSB_PDL_ENTRY();
    constexpr int V = Chunk<BF16>::kVec;
    constexpr int G = 32 / LPE;
    const int lane = threadIdx.x & 31;
    const int grp = lane / LPE, sub = lane % LPE;
    const int cpr = row_bytes >> 4;
    const int64_t nseg = m->n_dst * g.S;
    const int64_t E = seg_ptr[nseg];
    const int64_t pieces = (E + kSegCap - 1) / kSegCap;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t k = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; k < pieces; k += warps) {
        const int64_t pa = k * kSegCap, pb = min(E, pa + kSegCap);
        const int64_t qa = seg_find(seg_ptr, 0, nseg, pa, lane);
        const int64_t qb = seg_find(seg_ptr, qa, nseg, pb - 1, lane);
        for (int64_t q = qa;; q = qb) {
            const int64_t e0 = seg_ptr[q], e1 = seg_ptr[q + 1];
            const int64_t t0 = max(pa, e0 + kSegCap), t1 = min(pb, e1);
            if (t0 < t1) {
                const int64_t j = q / g.S;
                const int sl = (int)(q - j * g.S);
                const float inv = 1.f / (float)(e1 - e0);
                const uint4* prow = (t0 + lane < t1)
                    ? src_row<FEAT>(g, h, row_bytes, FEAT ? e_src_gid[t0 + lane] : (int64_t)e_src[t0 + lane], rowmap)
                    : nullptr;
                for (int c0 = 0; c0 < cpr; c0 += LPE) {
                    const int c = c0 + sub;
                    const bool cl = c < cpr;
                    float acc[V];
#pragma unroll
                    for (int v = 0; v < V; ++v) acc[v] = 0.f;
                    for (int64_t cb = t0; cb < t1; cb += 32) {
                        const uint4* pr = prow;
                        if (cb != t0)
                            pr = (cb + lane < t1) ? src_row<FEAT>(g, h, row_bytes,
                                                                  FEAT ? e_src_gid[cb + lane] : (int64_t)e_src[cb + lane],
                                                                  rowmap)
                                                  : nullptr;
                        const int cnt = (int)min((int64_t)32, t1 - cb);
                        for (int kk = 0; kk < cnt; kk += 4 * G) {
                            uint4 x[4];
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const int idx = kk + grp + G * u;
                                const uint64_t pu = __shfl_sync(0xffffffffu, (uint64_t)pr, idx & 31);
                                x[u] = make_uint4(0u, 0u, 0u, 0u);
                                if (cl && idx < cnt) x[u] = __ldg(reinterpret_cast<const uint4*>(pu) + c);
                            }
#pragma unroll
                            for (int u = 0; u < 4; ++u) chunk_acc<BF16>(acc, x[u]);
                        }
                    }
#pragma unroll
                    for (int o = LPE; o < 32; o <<= 1)
#pragma unroll
                        for (int v = 0; v < V; ++v) acc[v] += __shfl_xor_sync(0xffffffffu, acc[v], o);
                    if (cl && grp == 0) {
                        float* o = acat + j * lda + (int64_t)sl * d + (int64_t)c * V;
#pragma unroll
                        for (int v = 0; v < V; v += 4)
                            red_add_f4(o + v, make_float4(acc[v] * inv, acc[v + 1] * inv, acc[v + 2] * inv,
                                                          acc[v + 3] * inv));
                    }
                }
            }
            if (q == qb) break;
        }
    }
}

template <bool FEAT, bool BF16>
static gsb_status launch_heavy(cudaStream_t s, const GraphDev& g, const HopBufs& hb, const char* h, int row_bytes,
                               int d, float* acat, int64_t lda, const int32_t* rowmap) {
    const int cpr = row_bytes / 16;
    const int grid = kNumSMs * 8;
    if (cpr <= 8) {
        GSB_LAUNCH("rgcn_agg_heavy", (heavy_kernel<FEAT, BF16, 8>), grid, 256, 0, s, g, hb.meta, hb.seg_ptr, hb.e_src,
                   hb.e_src_gid, h, row_bytes, d, acat, lda, rowmap);
    } else if (cpr <= 16) {
        GSB_LAUNCH("rgcn_agg_heavy", (heavy_kernel<FEAT, BF16, 16>), grid, 256, 0, s, g, hb.meta, hb.seg_ptr, hb.e_src,
                   hb.e_src_gid, h, row_bytes, d, acat, lda, rowmap);
    } else {
        GSB_LAUNCH("rgcn_agg_heavy", (heavy_kernel<FEAT, BF16, 32>), grid, 256, 0, s, g, hb.meta, hb.seg_ptr, hb.e_src,
                   hb.e_src_gid, h, row_bytes, d, acat, lda, rowmap);
    }
    return GSB_OK;
}

// fanout: the hop's fanout (-1 = ALL); segments can exceed kSegCap only when it does
static gsb_status launch_agg(const char* name, bool feat, int dtype, cudaStream_t s, const GraphDev& g,
                             const HopBufs& hb, const void* h, int d, float* acat, int64_t lda, const int32_t* rowmap,
                             int fanout) {
    const int grid = grid_for(hb.cap_dst * 32, 256, kNumSMs * GSB_AGG_BPS);
    const int rb = d * dtype_size(dtype);
    const char* hc = static_cast<const char*>(h);
    const bool heavy = fanout < 0 || fanout > kSegCap;
    const int64_t cap = heavy ? kSegCap : INT64_MAX;
    gsb_status st;
    // segment-parallel kernel for hidden-layer inputs (layer >= 1: 10.0 vs 15.1 us under ncu on the
    // mag step); the layer-0 feature gather keeps the warp-per-row kernel, whose per-warp
    // address resolution beats the per-lane one there (profiles/round2_agg_ab.md).  GSB_AGG=warp /
    // seg forces either (A/B).  32-byte lanes: rows of 4..32 such chunks, 32-B aligned.
    const char* am = getenv("GSB_AGG");
    static const int agg_mode = !am ? 0 : (strcmp(am, "warp") == 0 ? 1 : (strcmp(am, "seg") == 0 ? 2 : 0));
    const bool want_seg = agg_mode == 2 || (agg_mode == 0 && !feat);
    const bool use_seg = want_seg && rb % 32 == 0 && rb / 32 >= 4 && rb / 32 <= 32 && d % 4 == 0 &&
                         (feat || (reinterpret_cast<uintptr_t>(h) & 31) == 0);
    if (use_seg) {
        if (feat)
            st = dtype == GSB_BF16 ? launch_agg_seg<true, true>(name, s, g, hb, hc, rb, d, acat, lda, rowmap, cap)
                                   : launch_agg_seg<true, false>(name, s, g, hb, hc, rb, d, acat, lda, rowmap, cap);
        else
            st = dtype == GSB_BF16 ? launch_agg_seg<false, true>(name, s, g, hb, hc, rb, d, acat, lda, rowmap, cap)
                                   : launch_agg_seg<false, false>(name, s, g, hb, hc, rb, d, acat, lda, rowmap, cap);
    } else if (feat)
        st = dtype == GSB_BF16 ? launch_agg_lpe<true, true>(name, grid, s, g, hb, hc, rb, d, acat, lda, rowmap, cap)
                               : launch_agg_lpe<true, false>(name, grid, s, g, hb, hc, rb, d, acat, lda, rowmap, cap);
    else
        st = dtype == GSB_BF16 ? launch_agg_lpe<false, true>(name, grid, s, g, hb, hc, rb, d, acat, lda, rowmap, cap)
                               : launch_agg_lpe<false, false>(name, grid, s, g, hb, hc, rb, d, acat, lda, rowmap, cap);
    if (st != GSB_OK || !heavy) return st;
    if (feat)
        return dtype == GSB_BF16 ? launch_heavy<true, true>(s, g, hb, hc, rb, d, acat, lda, rowmap)
                                 : launch_heavy<true, false>(s, g, hb, hc, rb, d, acat, lda, rowmap);
    return dtype == GSB_BF16 ? launch_heavy<false, true>(s, g, hb, hc, rb, d, acat, lda, rowmap)
                             : launch_heavy<false, false>(s, g, hb, hc, rb, d, acat, lda, rowmap);
}

// ------------------------------------------------------------------------------------
// backward scatter: dh_src[u] += dA[j, s] / c_s(j) per sampled edge; dh_src[self] += dA[j, S_t]
// ------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) scatter_kernel(GraphDev g, const HopMeta* __restrict__ m,
                                                      const int64_t* __restrict__ seg_ptr,
                                                      const int32_t* __restrict__ e_src, const float* __restrict__ dA,
                                                      int64_t lda, int d, float* __restrict__ dh) {
    GSB_PDL_ENTRY();
    const int lane = threadIdx.x & 31;
    const int S = g.S;
    const int64_t n = m->n_dst;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int d4 = d >> 2;
    for (int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; j < n; j += warps) {
        int t = 0;
        for (int k = 1; k < g.T; ++k) t += (j >= m->dst_off[k]) ? 1 : 0;
        const int St = g.n_slots[t];
        const float* row = dA + j * lda;
        for (int s = 0; s < St; ++s) {
            const int64_t e0 = seg_ptr[j * S + s], e1 = seg_ptr[j * S + s + 1];
            if (e1 == e0) continue;
            const float inv = 1.f / (float)(e1 - e0);
            for (int c = lane; c < d4; c += 32) {
                float4 v = reinterpret_cast<const float4*>(row + (int64_t)s * d)[c];
                v.x *= inv; v.y *= inv; v.z *= inv; v.w *= inv;
                for (int64_t e = e0; e < e1; ++e) red_add_f4(dh + (int64_t)e_src[e] * d + 4 * c, v);
            }
        }
        const int64_t self = m->src_off[t] + (j - m->dst_off[t]);
        for (int c = lane; c < d4; c += 32)
            red_add_f4(dh + self * d + 4 * c, reinterpret_cast<const float4*>(row + (int64_t)St * d)[c]);
    }
}

// Deterministic backward scatter through the block's transposed CSR (§8(a) a4): warp per src
// row u; its self term (u in the dst prefix: dA[j, S_t]) then its in-edges in ascending edge
// order, dA[j(e), s(e)] / c_s(j); one plain store per row (no atomics, no memset).
__global__ void __launch_bounds__(256) scatter_t_kernel(GraphDev g, const HopMeta* __restrict__ m,
                                                        const int32_t* __restrict__ t_seg,
                                                        const int32_t* __restrict__ t_ptr,
                                                        const int32_t* __restrict__ t_inv,
                                                        const float* __restrict__ dA, int64_t lda, int d,
                                                        float* __restrict__ dh) {
    GSB_PDL_ENTRY();
    const int lane = threadIdx.x & 31;
    const int S = g.S;
    const int64_t n_src = m->n_src;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int d4 = d >> 2;
    for (int64_t u = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; u < n_src; u += warps) {
        int t = 0;
        for (int k = 1; k < g.T; ++k) t += (u >= m->src_off[k]) ? 1 : 0;
        const int64_t local = u - m->src_off[t];
        float4 acc[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (local < m->dst_off[t + 1] - m->dst_off[t]) {     // u is dst row j's own row
            const int64_t j = m->dst_off[t] + local;
            const float4* row = reinterpret_cast<const float4*>(dA + j * lda + (int64_t)g.n_slots[t] * d);
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (lane + 32 * q < d4) acc[q] = row[lane + 32 * q];
        }
        const int32_t k0 = t_ptr[u], k1 = t_ptr[u + 1];
        for (int32_t kb = k0; kb < k1; kb += 4) {
            // up to 4 edges' gradient rows in flight, summed in ascending edge order
            float4 v[4][4];
            float inv[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                inv[e] = 0.f;
                if (kb + e < k1) {
                    const int32_t i = t_seg[kb + e];
                    const int64_t j = i / S;
                    const int s = i - (int)(j * S);
                    inv[e] = __int_as_float(t_inv[kb + e]);
                    const float4* row = reinterpret_cast<const float4*>(dA + j * lda + (int64_t)s * d);
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        v[e][q] = (lane + 32 * q < d4) ? row[lane + 32 * q] : make_float4(0.f, 0.f, 0.f, 0.f);
                }
            }
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (kb + e < k1)
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        acc[q].x += v[e][q].x * inv[e]; acc[q].y += v[e][q].y * inv[e];
                        acc[q].z += v[e][q].z * inv[e]; acc[q].w += v[e][q].w * inv[e];
                    }
        }
        float4* o = reinterpret_cast<float4*>(dh + u * d);
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (lane + 32 * q < d4) o[lane + 32 * q] = acc[q];
    }
}

// ------------------------------------------------------------------------------------
// softmax cross-entropy, warp per row; logits are overwritten by dlogits
// ------------------------------------------------------------------------------------
// Softmax CE, warp per row.  The batch mean is fused: every block writes the sum of its rows'
// losses to part[blockIdx]; the last block to finish (ticket) adds the partials in block order
// (deterministic) and resets the ticket for the next launch / graph replay.
__global__ void __launch_bounds__(256) ce_kernel(float* __restrict__ logits, int64_t n, int C, int64_t ldl,
                                                 const int32_t* __restrict__ labels,
                                                 const int64_t* __restrict__ seed_gid, int64_t base,
                                                 float* __restrict__ row_loss, float* __restrict__ part,
                                                 unsigned* __restrict__ ticket, float* __restrict__ loss) {
    GSB_PDL_ENTRY();
    __shared__ float wsum[8];
    __shared__ bool last;
    const int lane = threadIdx.x & 31;
    float mine = 0.f;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const float invn = 1.f / (float)n;
    constexpr int kR = 16;                         // row values held per lane (C <= 512)
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
        float* lg = logits + i * ldl;
        const int y = labels[seed_gid[i] - base];
        if (C <= 32 * kR) {   // one read of the row into registers
            float x[kR];
            float mx = -INFINITY, ly = 0.f;
#pragma unroll
            for (int k = 0; k < kR; ++k) {
                const int c = lane + 32 * k;
                x[k] = c < C ? lg[c] : -INFINITY;
                mx = fmaxf(mx, x[k]);
                if (c == y) ly = x[k];
            }
            for (int o = 16; o; o >>= 1) {
                mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                ly += __shfl_xor_sync(0xffffffffu, ly, o);     // one lane holds logit_y
            }
            float se = 0.f;
#pragma unroll
            for (int k = 0; k < kR; ++k) {
                const int c = lane + 32 * k;
                x[k] = c < C ? expf(x[k] - mx) : 0.f;
                se += x[k];
            }
            for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
            const float inv_se = 1.f / se;
#pragma unroll
            for (int k = 0; k < kR; ++k) {
                const int c = lane + 32 * k;
                if (c < C) lg[c] = (x[k] * inv_se - (c == y ? 1.f : 0.f)) * invn;
            }
            const float li = mx + logf(se) - ly;          // lse - logit_y
            if (lane == 0) row_loss[i] = li;
            mine += li;
            continue;
        }
        float mx = -INFINITY;
        for (int c = lane; c < C; c += 32) mx = fmaxf(mx, lg[c]);
        for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        float se = 0.f;
        for (int c = lane; c < C; c += 32) se += expf(lg[c] - mx);
        for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
        const float lse = mx + logf(se);
        const float li = lse - lg[y];
        if (lane == 0) row_loss[i] = li;
        mine += li;
        __syncwarp();
        for (int c = lane; c < C; c += 32) lg[c] = (expf(lg[c] - lse) - (c == y ? 1.f : 0.f)) * invn;
    }
    if (lane == 0) wsum[threadIdx.x >> 5] = mine;
    __syncthreads();
    if (threadIdx.x == 0) {
        float b = 0.f;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) b += wsum[w];
        part[blockIdx.x] = b;
        __threadfence();
        last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
    }
    __syncthreads();
    if (last && threadIdx.x < 32) {   // one warp adds the block partials (fixed order per lane)
        __threadfence();
        float tot = 0.f;
        for (unsigned b = threadIdx.x; b < gridDim.x; b += 32) tot += ((volatile float*)part)[b];
        for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        if (threadIdx.x == 0) {
            *loss = tot / (float)n;
            *ticket = 0u;
        }
    }
}

// ------------------------------------------------------------------------------------
// NC decoder, fused (SIMT fp32): north_star puts the tensor cores on the per-relation GEMMs
// only; the decoder's three [S0 x d] x [d x C] products (S0 = 1024, C = 349: 92 MFLOP each)
// are too small to amortise a tcgen05 pipeline (~10 us of fixed cost per launch).  Kernel 1,
// one CTA per TR seed rows: logits = h Wc + bc (thread per class column, Wc rows coalesced),
// softmax-CE per row (warp per row; loss, dlogits = (softmax - 1_y) / n), dh = dlogits Wc^T
// (warp per 1/8 of the hidden columns, lanes over classes, warp reductions), and the batch
// mean through per-block partials + a last-block ticket (deterministic order).  Kernel 2:
// dWc = h^T dlogits and dbc over row chunks (k-tile x row-chunk blocks, red.add).
// ------------------------------------------------------------------------------------
constexpr int kNcTR = 8;       // seed rows per CTA (one warp per row in the softmax)

__global__ void __launch_bounds__(256) nc_fused_kernel(const float* __restrict__ h, int64_t n, int d,
                                                       const float* __restrict__ Wc, const float* __restrict__ bc,
                                                       int C, int64_t ldl, const int32_t* __restrict__ labels,
                                                       const int64_t* __restrict__ seed_gid, int64_t base,
                                                       float* __restrict__ dl_out, float* __restrict__ row_loss,
                                                       float* __restrict__ part, unsigned* __restrict__ ticket,
                                                       float* __restrict__ loss, float* __restrict__ dh) {
    GSB_PDL_ENTRY();
    extern __shared__ float sm[];
    float* sh = sm;                          // [TR][d]   seed rows
    float* sl = sm + kNcTR * d;              // [TR][ldl] logits, then dlogits
    __shared__ float wsum[8];
    __shared__ bool last;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float invn = 1.f / (float)n;
    float mine = 0.f;
    const int64_t tiles = (n + kNcTR - 1) / kNcTR;
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const int64_t r0 = tile * kNcTR;
        const int nr = (int)min((int64_t)kNcTR, n - r0);
        for (int x = tid; x < kNcTR * d; x += blockDim.x) {
            const int r = x / d, k = x - r * d;
            sh[x] = r < nr ? h[(r0 + r) * d + k] : 0.f;
        }
        __syncthreads();
        // logits: thread per class column, Wc row k read coalesced across the block
        for (int c = tid; c < C; c += blockDim.x) {
            float acc[kNcTR];
            const float b = __ldg(bc + c);
#pragma unroll
            for (int r = 0; r < kNcTR; ++r) acc[r] = b;
#pragma unroll 4
            for (int k = 0; k < d; k += 4) {     // d % 32 == 0; 16-B smem broadcasts of the rows
                const float w0 = __ldg(Wc + (int64_t)k * C + c), w1 = __ldg(Wc + (int64_t)(k + 1) * C + c);
                const float w2 = __ldg(Wc + (int64_t)(k + 2) * C + c), w3 = __ldg(Wc + (int64_t)(k + 3) * C + c);
#pragma unroll
                for (int r = 0; r < kNcTR; ++r) {
                    const float4 x = *reinterpret_cast<const float4*>(sh + r * d + k);
                    acc[r] += x.x * w0 + x.y * w1 + x.z * w2 + x.w * w3;
                }
            }
#pragma unroll
            for (int r = 0; r < kNcTR; ++r) sl[r * ldl + c] = acc[r];
        }
        __syncthreads();
        // softmax-CE: warp r owns row r
        if (warp < nr) {
            const int r = warp;
            const int64_t i = r0 + r;
            float* row = sl + r * ldl;
            const int y = labels[seed_gid[i] - base];
            float mx = -INFINITY;
            for (int c = lane; c < C; c += 32) mx = fmaxf(mx, row[c]);
            for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            float se = 0.f;
            for (int c = lane; c < C; c += 32) se += expf(row[c] - mx);
            for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
            const float lse = mx + logf(se);
            const float li = lse - row[y];
            __syncwarp();
            for (int c = lane; c < C; c += 32) {
                const float g = (expf(row[c] - lse) - (c == y ? 1.f : 0.f)) * invn;
                row[c] = g;
                dl_out[i * ldl + c] = g;
            }
            if (lane == 0) {
                row_loss[i] = li;
                mine += li;
            }
        } else if (warp < kNcTR) {
            for (int c = lane; c < C; c += 32) sl[warp * ldl + c] = 0.f;
        }
        __syncthreads();
        // dh = dlogits Wc^T: warp w owns hidden columns k = w, w + 8, ...; lanes over classes
        for (int k = warp; dh && k < d; k += 8) {
            float acc[kNcTR];
#pragma unroll
            for (int r = 0; r < kNcTR; ++r) acc[r] = 0.f;
            const float* wk = Wc + (int64_t)k * C;
#pragma unroll 4
            for (int c = lane; c < C; c += 32) {
                const float w = __ldg(wk + c);
#pragma unroll
                for (int r = 0; r < kNcTR; ++r) acc[r] += sl[r * ldl + c] * w;
            }
#pragma unroll
            for (int r = 0; r < kNcTR; ++r) {
                float v = acc[r];
                for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                if (lane == 0 && r < nr) dh[(r0 + r) * d + k] = v;
            }
        }
        __syncthreads();
    }
    // batch mean: block partial, the last block adds the partials in block order
    if (lane == 0) wsum[warp] = mine;
    __syncthreads();
    if (tid == 0) {
        float b = 0.f;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) b += wsum[w];
        part[blockIdx.x] = b;
        __threadfence();
        last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
    }
    __syncthreads();
    if (last && tid < 32) {
        __threadfence();
        float tot = 0.f;
        for (unsigned b = tid; b < gridDim.x; b += 32) tot += ((volatile float*)part)[b];
        for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
        if (tid == 0) {
            *loss = tot / (float)n;
            *ticket = 0u;
        }
    }
}

// dWc[k][c] += sum over a row chunk of h[r][k] * dl[r][c] (k-tile of 16 x row chunk per block;
// thread per class column), dbc[c] += sum over the chunk of dl[r][c] (k-tile 0 blocks)
constexpr int kNcKT = 16, kNcRC = 128;
__global__ void __launch_bounds__(256) nc_dwc_kernel(const float* __restrict__ h, int64_t n, int d,
                                                     const float* __restrict__ dl, int64_t ldl, int C,
                                                     float* __restrict__ dWc, float* __restrict__ dbc) {
    GSB_PDL_ENTRY();
    __shared__ float shk[kNcRC][kNcKT];
    const int nkt = (d + kNcKT - 1) / kNcKT;
    const int kt = blockIdx.x % nkt;
    const int64_t r0 = (int64_t)(blockIdx.x / nkt) * kNcRC;
    const int k0 = kt * kNcKT;
    const int nr = (int)min((int64_t)kNcRC, n - r0);
    for (int x = threadIdx.x; x < kNcRC * kNcKT; x += blockDim.x) {
        const int r = x / kNcKT, k = x - r * kNcKT;
        shk[r][k] = (r < nr && k0 + k < d) ? h[(r0 + r) * d + k0 + k] : 0.f;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
        float acc[kNcKT];
#pragma unroll
        for (int k = 0; k < kNcKT; ++k) acc[k] = 0.f;
        float sb = 0.f;
#pragma unroll 8
        for (int r = 0; r < nr; ++r) {
            const float g = dl[(r0 + r) * ldl + c];
            sb += g;
#pragma unroll
            for (int k = 0; k < kNcKT; ++k) acc[k] += shk[r][k] * g;
        }
#pragma unroll
        for (int k = 0; k < kNcKT; ++k)
            if (k0 + k < d) atomicAdd(dWc + (int64_t)(k0 + k) * C + c, acc[k]);
        if (kt == 0) atomicAdd(dbc + c, sb);
    }
}

__global__ void __launch_bounds__(1024) mean_kernel(const float* __restrict__ x, int64_t n, float* __restrict__ out) {
    GSB_PDL_ENTRY();
    __shared__ float sm[32];
    float s = 0.f;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += x[i];
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = (threadIdx.x < (blockDim.x >> 5)) ? sm[threadIdx.x] : 0.f;
        for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) *out = s / (float)n;
    }
}

// dZ = dh * 1[h > 0] in place (ReLU backward, ReLU'(0) = 0), rows = device dst count
__global__ void __launch_bounds__(256) relu_bwd_kernel(const HopMeta* __restrict__ m, float* __restrict__ dh,
                                                       const float* __restrict__ h, int d) {
    GSB_PDL_ENTRY();
    const int64_t n4 = m->n_dst * (int64_t)d / 4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        float4 g = reinterpret_cast<float4*>(dh)[i];
        const float4 x = __ldg(reinterpret_cast<const float4*>(h) + i);
        g.x = x.x > 0.f ? g.x : 0.f; g.y = x.y > 0.f ? g.y : 0.f;
        g.z = x.z > 0.f ? g.z : 0.f; g.w = x.w > 0.f ? g.w : 0.f;
        reinterpret_cast<float4*>(dh)[i] = g;
    }
}

// zero the first n_dst (device count) rows of a [rows][w] fp32 output before split-K
// partials are red.added into it: a capacity-sized memset would write past a caller buffer
// that holds only the live rows (e.g. one chunk of a full-graph table)
__global__ void __launch_bounds__(256) zero_rows_kernel(const HopMeta* __restrict__ m, float* __restrict__ p,
                                                        int64_t w) {
    GSB_PDL_ENTRY();
    const int64_t n = m->n_dst * w;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        p[i] = 0.f;
}

static const char* lname(const char* base, int layer) {
    static const char* names[][4] = {
        {"rgcn_agg_l0", "rgcn_agg_l1", "rgcn_agg_l2", "rgcn_agg_l3"},
        {"rgcn_gemm_fwd_l0", "rgcn_gemm_fwd_l1", "rgcn_gemm_fwd_l2", "rgcn_gemm_fwd_l3"},
        {"rgcn_gemm_dW_l0", "rgcn_gemm_dW_l1", "rgcn_gemm_dW_l2", "rgcn_gemm_dW_l3"},
        {"rgcn_gemm_dA_l0", "rgcn_gemm_dA_l1", "rgcn_gemm_dA_l2", "rgcn_gemm_dA_l3"},
        {"rgcn_scatter_l0", "rgcn_scatter_l1", "rgcn_scatter_l2", "rgcn_scatter_l3"},
        {"relu_bwd_l0", "relu_bwd_l1", "relu_bwd_l2", "relu_bwd_l3"}};
    int k = 0;
    const char* keys[] = {"rgcn_agg", "rgcn_gemm_fwd", "rgcn_gemm_dW", "rgcn_gemm_dA", "rgcn_scatter", "relu_bwd"};
    for (; k < 6; ++k)
        if (strcmp(base, keys[k]) == 0) break;
    return (k < 6 && layer >= 0 && layer < 4) ? names[k][layer] : base;
}

static RowGroups layer_groups(const Blocks* B, const void* arena, int layer) {
    RowGroups rg;
    memset(&rg, 0, sizeof(rg));
    const GraphDev& g = B->g->dev;
    rg.meta = at<HopMeta>(const_cast<void*>(arena), B->off_meta[B->hop_of_layer(layer)]);
    rg.G = g.T;
    for (int t = 0; t < g.T; ++t) {
        rg.ks[t] = g.n_slots[t] + 1;
        for (int s = 0; s < g.n_slots[t]; ++s) rg.slot_w[t][s] = g.slot_etype[t][s];
        rg.slot_w[t][g.n_slots[t]] = g.R;  // W_self
    }
    return rg;
}

static RowGroups single_group(int64_t M) {
    RowGroups rg;
    memset(&rg, 0, sizeof(rg));
    rg.meta = nullptr;
    rg.M = M;
    rg.G = 1;
    rg.ks[0] = 1;
    rg.slot_w[0][0] = 0;
    return rg;
}


}  // namespace gsb

using namespace gsb;

extern "C" {

gsb_status gsb_layer_acat_floats(gsb_blocks_t b, int32_t layer, int32_t d_in, int64_t* n_floats) {
    Blocks* B = reinterpret_cast<Blocks*>(b);
    GSB_CHECK_ARG(B && n_floats && layer >= 0 && layer < B->L && d_in > 0, "bad argument");
    *n_floats = B->cap_dst[B->hop_of_layer(layer)] * (int64_t)(B->g->dev.S + 1) * d_in;
    return GSB_OK;
}

gsb_status gsb_rgcn_layer_fwd(gsb_blocks_t b, const void* arena, int32_t layer, const float* h_src, int32_t d_in,
                              const float* W, const float* bias, int32_t d_out, int32_t relu, float* h_dst,
                              float* acat, void* stream) {
    return gsb_rgcn_layer_fwd_ex(b, arena, layer, h_src, GSB_F32, nullptr, d_in, W, bias, d_out, relu, h_dst, acat,
                                 stream);
}

gsb_status gsb_rgcn_layer_agg(gsb_blocks_t b, const void* arena, int32_t layer, const void* h_src, int32_t h_dtype,
                              const int32_t* rowmap, int32_t d_in, float* acat, void* stream) {
    Blocks* B = reinterpret_cast<Blocks*>(b);
    GSB_CHECK_ARG(B && arena && acat, "null argument");
    GSB_CHECK_ARG(h_src || layer == 0, "h_src may be NULL only for layer 0 (features read by gid)");
    GSB_CHECK_ARG(layer >= 0 && layer < B->L, "layer %d out of range", layer);
    GSB_CHECK_ARG(d_in > 0 && d_in % BK == 0, "d_in %d must be a multiple of %d", d_in, BK);
    GSB_CHECK_ARG(!rowmap || h_src, "rowmap needs h_src");
    cudaStream_t s = (cudaStream_t)stream;
    const int h = B->hop_of_layer(layer);
    HopBufs hb = B->hop(h, const_cast<void*>(arena));
    const GraphDev& g = B->g->dev;
    const int64_t lda = (int64_t)(g.S + 1) * d_in;
    if (h_src) {
        GSB_CHECK_ARG(dtype_size(h_dtype) > 0, "h_dtype %d not GSB_F32 / GSB_BF16", h_dtype);
        return launch_agg(lname("rgcn_agg", layer), false, h_dtype, s, g, hb, h_src, d_in, acat, lda, rowmap,
                          B->fanout[layer]);
    }
    GSB_CHECK_ARG(g.feat_dim == d_in, "layer 0 with features: d_in %d != feature dim %d", d_in, g.feat_dim);
    for (int t = 0; t < g.T; ++t) GSB_CHECK_ARG(g.feat[t], "features of ntype %d not registered", t);
    return launch_agg(lname("rgcn_agg", layer), true, g.feat_dtype, s, g, hb, nullptr, d_in, acat, lda, nullptr,
                      B->fanout[layer]);
}

gsb_status gsb_rgcn_layer_gemm(gsb_blocks_t b, const void* arena, int32_t layer, const float* acat, int32_t d_in,
                               const float* W, const float* bias, int32_t d_out, int32_t relu, float* h_dst,
                               void* stream) {
    Blocks* B = reinterpret_cast<Blocks*>(b);
    GSB_CHECK_ARG(B && arena && W && h_dst && acat, "null argument");
    GSB_CHECK_ARG(layer >= 0 && layer < B->L, "layer %d out of range", layer);
    GSB_CHECK_ARG(d_in > 0 && d_in % BK == 0, "d_in %d must be a multiple of %d", d_in, BK);
    GSB_CHECK_ARG(d_out > 0 && d_out % 4 == 0, "d_out %d must be a multiple of 4", d_out);
    cudaStream_t s = (cudaStream_t)stream;
    const int h = B->hop_of_layer(layer);
    HopBufs hb = B->hop(h, const_cast<void*>(arena));
    const GraphDev& g = B->g->dev;
    const int64_t lda = (int64_t)(g.S + 1) * d_in;
    RowGroups rg = layer_groups(B, arena, layer);
    UProb P{};
    P.rg = rg; P.A = acat; P.lda = lda; P.B = W; P.ldb = d_out; P.bslot = (int64_t)d_in * d_out;
    P.relu = relu; P.d_in = d_in; P.N = d_out; P.C = h_dst; P.ldc = d_out; P.bias = bias;
    const int64_t tiles = (ceil_div(hb.cap_dst, 128) + g.T) * ceil_div(d_out, 128);
    P.ksplit = choose_ksplit(tiles, (g.S + 1) * (d_in / 32), !relu);
    if (P.ksplit > 1)
        GSB_LAUNCH("zero_rows", zero_rows_kernel, grid_for(hb.cap_dst * d_out, 256, kNumSMs * 4), 256, 0, s, hb.meta,
                   h_dst, (int64_t)d_out);
    return launch_gemm_v<UMMA_NN>(lname("rgcn_gemm_fwd", layer), P, tiles, hb.cap_dst, lda, (int64_t)(g.R + 1) * d_in,
                                d_out, s);
}

gsb_status gsb_rgcn_layer_fwd_ex(gsb_blocks_t b, const void* arena, int32_t layer, const void* h_src, int32_t h_dtype,
                                 const int32_t* rowmap, int32_t d_in, const float* W, const float* bias, int32_t d_out,
                                 int32_t relu, float* h_dst, float* acat, void* stream) {
    GSB_CHECK_ARG(W && h_dst, "null argument");
    gsb_status st = gsb_rgcn_layer_agg(b, arena, layer, h_src, h_dtype, rowmap, d_in, acat, stream);
    if (st != GSB_OK) return st;
    return gsb_rgcn_layer_gemm(b, arena, layer, acat, d_in, W, bias, d_out, relu, h_dst, stream);
}

gsb_status gsb_rgcn_layer_bwd(gsb_blocks_t b, const void* arena, int32_t layer, const float* h_dst,
                              float* dh_dst, const float* W, const float* acat, int32_t d_in, int32_t d_out,
                              int32_t relu, float* dW, float* db, float* dh_src, float* dacat_ws, void* stream) {
    Blocks* B = reinterpret_cast<Blocks*>(b);
    GSB_CHECK_ARG(B && arena && dh_dst && W && acat && dW && db, "null argument");
    GSB_CHECK_ARG(!relu || h_dst, "relu backward needs h_dst");
    GSB_CHECK_ARG(!dh_src || dacat_ws, "dh_src needs dacat_ws");
    GSB_CHECK_ARG(layer >= 0 && layer < B->L, "layer %d out of range", layer);
    GSB_CHECK_ARG(d_in > 0 && d_in % BK == 0 && d_out > 0 && d_out % 4 == 0, "bad dims");
    cudaStream_t s = (cudaStream_t)stream;
    const GraphDev& g = B->g->dev;
    const int h = B->hop_of_layer(layer);
    HopBufs hb = B->hop(h, const_cast<void*>(arena));
    const int64_t lda = (int64_t)(g.S + 1) * d_in;
    RowGroups rg = layer_groups(B, arena, layer);
    // row chunks of the weight gradient sized so the (type, slot, chunk) items cover ~2 waves of SMs
    const int64_t rows = hb.cap_dst;
    int rpc = (int)std::max<int64_t>(64, std::min<int64_t>(2048, ceil_div(rows * (g.S + 1), 2 * kNumSMs)));
    rpc = (rpc + 31) / 32 * 32;
    UProb Pw{};
    Pw.rg = rg; Pw.A = acat; Pw.lda = lda; Pw.B = dh_dst; Pw.ldb = d_out;
    Pw.d_in = d_in; Pw.N = d_out; Pw.C = dW; Pw.ldc = d_out; Pw.bslot = (int64_t)d_in * d_out; Pw.db = db;
    Pw.rows_per_chunk = rpc;
    // dZ = dh * 1[h > 0] once in place before the GEMMs (folding the mask into the weight-gradient
    // GEMM's B split measured slower: dW_l0 29.3 -> 33.3 us, profiles/round2_gemm_tma3.md)
    if (relu) {
        GSB_LAUNCH(lname("relu_bwd", layer), relu_bwd_kernel, grid_for(hb.cap_dst * d_out / 4, 256, kNumSMs * 8), 256, 0, s,
                   hb.meta, dh_dst, h_dst, d_out);
    }
    // the weight gradient runs on the side stream, overlapping dA + scatter (joined below)
    cudaStream_t s_main = s;
    if (dh_src) s = fork_begin(s_main);
    GSB_CUDA(cudaMemsetAsync(dW, 0, sizeof(float) * (size_t)(g.R + 1) * d_in * d_out, s));
    GSB_CUDA(cudaMemsetAsync(db, 0, sizeof(float) * (size_t)d_out, s));
    {
        int64_t items = (ceil_div(rows, rpc) + g.T) * (g.S + 1) * ceil_div(d_in, 128) * ceil_div(d_out, 128);
        gsb_status st = launch_gemm_v<UMMA_TN>(lname("rgcn_gemm_dW", layer), Pw, items, hb.cap_dst, lda, hb.cap_dst,
                                               d_out, s);
        if (st != GSB_OK) return st;
    }
    cudaStream_t s_side = s;
    s = s_main;
    if (dh_src) {
        UProb P{};
        P.rg = rg; P.A = dh_dst; P.lda = d_out; P.B = W; P.ldb = d_out;
        P.bslot = (int64_t)d_in * d_out; P.d_in = d_in; P.N = d_out; P.C = dacat_ws; P.ldc = lda;
        const int64_t tiles = (ceil_div(hb.cap_dst, 128) + g.T) * ceil_div(d_in, 128) * (g.S + 1);
        P.ksplit = choose_ksplit(tiles, (d_out + 31) / 32, true);
        if (P.ksplit > 1) GSB_CUDA(cudaMemsetAsync(dacat_ws, 0, sizeof(float) * (size_t)hb.cap_dst * lda, s));
        gsb_status st = launch_gemm_v<UMMA_NT>(lname("rgcn_gemm_dA", layer), P, tiles, hb.cap_dst, d_out,
                                             (int64_t)(g.R + 1) * d_in, d_out, s);
        if (st != GSB_OK) return st;
        // deterministic gather scatter through the transposed CSR when the sampler built it
        // (GSB_TCSR=1; bit-reproducible but slower here: profiles/round2_decoder_scatter.md)
        if (hb.t_ptr && d_in <= 512 && d_in % 4 == 0) {
            GSB_LAUNCH(lname("rgcn_scatter", layer), scatter_t_kernel, grid_for(hb.cap_src * 32, 256, kNumSMs * 8), 256,
                       0, s, g, hb.meta, hb.t_key, hb.t_ptr, hb.t_val, dacat_ws, lda, d_in, dh_src);
        } else {
            GSB_CUDA(cudaMemsetAsync(dh_src, 0, sizeof(float) * (size_t)hb.cap_src * d_in, s));
            GSB_LAUNCH(lname("rgcn_scatter", layer), scatter_kernel, grid_for(hb.cap_dst * 32, 256, kNumSMs * 8), 256, 0,
                       s, g, hb.meta, hb.seg_ptr, hb.e_src, dacat_ws, lda, d_in, dh_src);
        }
    }
    return fork_end(s_main, s_side);
}

gsb_status gsb_gemm_trace(uint64_t* out, int32_t n) {
    GSB_CHECK_ARG(out && n > 0 && n <= 4 * TG_TRACE, "bad argument");
    GSB_CUDA(cudaMemcpyFromSymbol(out, g_gemm_trace, sizeof(uint64_t) * n));
    return GSB_OK;
}

gsb_status gsb_gemm(int32_t mode, const float* A, int64_t lda, const float* B, int64_t ldb, int64_t M, int32_t N,
                    int32_t K, float* C, int64_t ldc, void* stream) {
    GSB_CHECK_ARG(A && B && C && M >= 1 && N >= 1 && K >= 1, "bad argument");
    cudaStream_t s = (cudaStream_t)stream;
    UProb P{};
    P.rg = single_group(M);
    P.A = A; P.lda = lda; P.B = B; P.ldb = ldb; P.C = C; P.ldc = ldc;
    if (mode == 0) {            // C[M][N] = A[M][K] B[K][N]
        GSB_CHECK_ARG(K % 32 == 0, "NN needs K %% 32 == 0");
        P.d_in = K; P.N = N;
        return launch_gemm_v<UMMA_NN>("gemm_nn", P, ceil_div(M, 128) * ceil_div(N, 128), M, K, K, N, s);
    } else if (mode == 1) {     // C[M][K] = A[M][N] B[K][N]^T
        P.d_in = K; P.N = N;
        return launch_gemm_v<UMMA_NT>("gemm_nt", P, ceil_div(M, 128) * ceil_div(K, 128), M, N, K, N, s);
    } else if (mode == 2) {     // C[K][N] += A[M][K]^T B[M][N]
        P.d_in = K; P.N = N; P.rows_per_chunk = 128;
        return launch_gemm_v<UMMA_TN>("gemm_tn", P, ceil_div(M, 128) * ceil_div(K, 128) * ceil_div(N, 128), M, K, M,
                                    N, s);
    }
    set_error("mode %d not in {0,1,2}", mode);
    return GSB_EINVAL;
}

// dWc = h^T dlogits, dbc = column sums of dlogits (dlogits: what nc_ce / nc_fused left in
// logits_ws); fused: the SIMT kernel of the GSB_NC=fused decoder, else the tcgen05 TN GEMM
__global__ void pad_copy_kernel(const float* __restrict__ src, int64_t ld, int64_t rows, int cols,
                                float* __restrict__ dst) {
    GSB_PDL_ENTRY();
    const int64_t total = rows * cols;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / cols;
        dst[i] = src[r * ld + (i - r * cols)];
    }
}

// pad_ws (optional, [d][ldl] fp32): when C's rows are not 16-B multiples, the TN GEMM
// reduce-adds its row-chunk partials into pad_ws with TMA (instead of 16k per-thread atomics
// per CTA into the unaligned dWc) and one copy kernel writes dWc
static gsb_status nc_dw(const float* h, int64_t n, int32_t d, const float* logits_ws, int64_t ldl, int32_t C,
                        float* dWc, float* dbc, bool fused, cudaStream_t s, float* pad_ws = nullptr) {
    const bool padded = !fused && pad_ws && ldl != C && (reinterpret_cast<uintptr_t>(pad_ws) & 15) == 0;
    float* dst = padded ? pad_ws : dWc;
    const int64_t ldd = padded ? ldl : C;
    GSB_CUDA(cudaMemsetAsync(dst, 0, sizeof(float) * (size_t)d * ldd, s));
    GSB_CUDA(cudaMemsetAsync(dbc, 0, sizeof(float) * (size_t)C, s));
    if (fused) {
        const int nkt = (d + kNcKT - 1) / kNcKT;
        GSB_LAUNCH("nc_dwc", nc_dwc_kernel, (int)(nkt * ((n + kNcRC - 1) / kNcRC)), 256, 0, s, h, n, d, logits_ws, ldl,
                   C, dWc, dbc);
        return GSB_OK;
    }
    UProb P{};
    P.rg = single_group(n);
    P.A = h; P.lda = d; P.B = logits_ws; P.ldb = ldl; P.d_in = d; P.N = C; P.C = dst; P.ldc = ldd;
    static const int rpc = getenv("GSB_DWC_RPC") ? atoi(getenv("GSB_DWC_RPC")) : 64;   // A/B knob
    P.bslot = 0; P.db = dbc; P.rows_per_chunk = rpc;
    gsb_status st = launch_gemm_v<UMMA_TN>("nc_gemm_dWc", P, ceil_div(n, rpc) * ceil_div(d, 128) * ceil_div(C, 128), n,
                                           d, n, C, s);
    if (st != GSB_OK || !padded) return st;
    GSB_LAUNCH("nc_dwc_copy", pad_copy_kernel, grid_for((int64_t)d * C, 256, kNumSMs * 2), 256, 0, s, pad_ws, ldl,
               (int64_t)d, C, dWc);
    return GSB_OK;
}

static bool nc_fused_mode() {   // read per call: tests switch it inside one process
    const char* e = getenv("GSB_NC");
    return e && strcmp(e, "fused") == 0;
}

gsb_status gsb_nc_loss_dw(const float* h, int64_t n, int32_t d, const float* logits_ws, int32_t C, float* dWc,
                          float* dbc, float* pad_ws, void* stream) {
    GSB_CHECK_ARG(h && logits_ws && dWc && dbc, "null argument");
    GSB_CHECK_ARG(n >= 1 && d > 0 && d % BK == 0 && C >= 1, "bad dims (d %% %d == 0 required)", BK);
    const int64_t ldl = (C + 3) / 4 * 4;
    const bool fused = nc_fused_mode() && sizeof(float) * (size_t)kNcTR * (d + ldl) <= 48 * 1024;
    return nc_dw(h, n, d, logits_ws, ldl, C, dWc, dbc, fused, (cudaStream_t)stream, pad_ws);
}

gsb_status gsb_nc_loss(const float* h, int64_t n, int32_t d, const float* Wc, const float* bc, int32_t C,
                       const int32_t* labels, const int64_t* seed_gid, int64_t label_gid_base, float* logits_ws,
                       float* row_loss_ws, float* loss, float* dh, float* dWc, float* dbc, void* stream) {
    GSB_CHECK_ARG(h && Wc && bc && labels && seed_gid && logits_ws && row_loss_ws && loss, "null argument");
    GSB_CHECK_ARG(n >= 1 && d > 0 && d % BK == 0 && C >= 1, "bad dims (d %% %d == 0 required)", BK);
    cudaStream_t s = (cudaStream_t)stream;
    RowGroups rg = single_group(n);
    const int64_t ldl = (C + 3) / 4 * 4;   // padded logits row (16-B aligned rows)
    // fused SIMT decoder: opt-in (GSB_NC=fused); measured slower than the tcgen05 GEMMs + CE on the
    // mag step (69.6 + 45.8 us vs 16.4 + 9.8 + 20.3 || 16.4 us, profiles/round2_decoder_scatter.md)
    const bool nc_fused = nc_fused_mode();
    const size_t fsm = sizeof(float) * (size_t)kNcTR * (d + ldl);
    if (nc_fused && fsm <= 48 * 1024) {
        float* part = row_loss_ws + ((n + 31) / 32) * 32;
        unsigned* ticket = reinterpret_cast<unsigned*>(part + kNumSMs * 4);
        const int grid = (int)std::min<int64_t>((n + kNcTR - 1) / kNcTR, kNumSMs * 4);
        GSB_LAUNCH("nc_fused", nc_fused_kernel, grid, 256, fsm, s, h, n, d, Wc, bc, C, ldl, labels, seed_gid,
                   label_gid_base, logits_ws, row_loss_ws, part, ticket, loss, dh);
        if (dWc || dbc) {
            GSB_CHECK_ARG(dWc && dbc, "dWc and dbc go together");
            return nc_dw(h, n, d, logits_ws, ldl, C, dWc, dbc, true, s);
        }
        return GSB_OK;
    }
    {
        UProb P{};
        P.rg = rg; P.A = h; P.lda = d; P.B = Wc; P.ldb = C; P.bslot = 0; P.d_in = d; P.N = C; P.C = logits_ws;
        P.ldc = ldl; P.bias = bc;
        const int64_t tiles = ceil_div(n, 128) * ceil_div(C, 128);
        P.ksplit = choose_ksplit(tiles, d / 32, true);
        if (P.ksplit > 1) GSB_CUDA(cudaMemsetAsync(logits_ws, 0, sizeof(float) * (size_t)n * ldl, s));
        gsb_status st = launch_gemm_v<UMMA_NN>("nc_logits", P, tiles, n, d, d, C, s);
        if (st != GSB_OK) return st;
    }
    {
        // fused batch mean: partials and the ticket word live in row_loss_ws after the n row
        // losses (caller-owned scratch of n + 640 floats, zero-filled before first use)
        const int grid = grid_for(n * 32, 256, kNumSMs * 4);
        float* part = row_loss_ws + ((n + 31) / 32) * 32;
        unsigned* ticket = reinterpret_cast<unsigned*>(part + kNumSMs * 4);
        GSB_LAUNCH("nc_ce", ce_kernel, grid, 256, 0, s, logits_ws, n, C, ldl, labels, seed_gid, label_gid_base,
                   row_loss_ws, part, ticket, loss);
    }
    cudaStream_t s_main = s;
    if (dWc && dh) s = fork_begin(s_main);   // dWc on the side stream, overlapping dh
    if (dWc || dbc) {
        GSB_CHECK_ARG(dWc && dbc, "dWc and dbc go together");
        gsb_status st = nc_dw(h, n, d, logits_ws, ldl, C, dWc, dbc, false, s);
        if (st != GSB_OK) return st;
    }
    cudaStream_t s_side = s;
    s = s_main;
    if (dh) {
        UProb P{};
        P.rg = rg; P.A = logits_ws; P.lda = ldl; P.B = Wc; P.ldb = C; P.bslot = 0; P.d_in = d; P.N = C; P.C = dh;
        P.ldc = d;
        const int64_t tiles = ceil_div(n, 128) * ceil_div(d, 128);
        P.ksplit = choose_ksplit(tiles, (C + 31) / 32, true);
        if (P.ksplit > 1) GSB_CUDA(cudaMemsetAsync(dh, 0, sizeof(float) * (size_t)n * d, s));
        gsb_status st = launch_gemm_v<UMMA_NT>("nc_gemm_dh", P, tiles, n, C, d, C, s);
        if (st != GSB_OK) return st;
    }
    return fork_end(s_main, s_side);
}

}  // extern "C"
