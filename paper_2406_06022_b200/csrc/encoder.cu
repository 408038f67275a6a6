// encoder.cu -- input encoder ("node input encoders", P:L156
// featureless nodes) over the input rows of a sampled mini-batch (layer-0 src rows):
//   H0[i] = F_t[local(i)] W_t      ntype t with a projection (bf16 rows, dim_t -> d_out)
//   H0[i] = F_t[local(i)]          frozen table (dim_t == d_out), widened to fp32
// and its weight gradient dW_t = sum_{i of type t} F_t[local(i)]^T dH0[i].
//
// Both products run on tcgen05 kind::f16 (bf16 operands, fp32 accumulation in TMEM).  The
// feature rows are exact bf16; the fp32 operand (W_t forward, dH0 backward) is split into
// bf16 hi + lo (hi = bf16(x), lo = bf16(x - hi); |x - hi - lo| <= 2^-17 |x|) and both halves
// are multiplied, so the products keep fp32-class accuracy.  Feature rows are
// gathered by gid straight into the swizzled operand panels with cp.async (no X0 buffer).
// Contract: include/gsb.h "Input encoder".
#include <cuda_bf16.h>

#include <cuda.h>

#include "gemm_tma.cuh"
#include "gsb_internal.cuh"
#include "umma.cuh"

namespace gsb {

using umma::cp16;
using umma::cp4;
using umma::cp_commit;
using umma::cp_wait;

constexpr int EN_PANEL = 16384;            // 128 x 64 bf16 (fwd) / 128 MN x 64 K bf16 (dW)
// decoupled rings: the gathered A panels (HBM-latency bound, deep ring) and the dense B panels
// (W^T / dH0 hi + lo by TMA, mostly L2 hits, shallow ring)
#ifndef GSB_ENC_AF
#define GSB_ENC_AF 8      // forward: A stages (B = W^T panels, 2 stages: L2 hits)
#endif
#ifndef GSB_ENC_AB
#define GSB_ENC_AB 4      // weight gradient: A stages (B = dH0 panels, 4 stages)
#endif
template <bool BWD>
struct EnRing {
    static constexpr int A = BWD ? GSB_ENC_AB : GSB_ENC_AF;
    static constexpr int B = (192 - 16 * A) / 32;
};
constexpr int EN_B_STAGE = 2 * EN_PANEL;   // B_hi, B_lo
constexpr int EN_SMEM = 192 * 1024 + 1024;

struct EncDev {
    int T, d_out;
    int proj[kMaxT];
    int dim[kMaxT];
    const __nv_bfloat16* wt_hi[kMaxT];     // [d_out][dim_t] (W_t transposed: K-major B operand)
    const __nv_bfloat16* wt_lo[kMaxT];
    const __nv_bfloat16* d_hi;             // [rows][d_out] split dH0 (backward)
    const __nv_bfloat16* d_lo;
};

struct EncOut {
    float* dW[kMaxT];                      // backward: dW_t [dim_t][d_out] (accumulated)
};

// TMA maps of the B operand (use = 1): forward: W_t^T hi / lo per projected type, [d_out][dim_t]
// bf16, box {64, 128} SWIZZLE_128B (= the K-major kmaj16 panel layout); backward: dH0 hi / lo
// [rows][d_out] bf16 in [0], box {64, 64} SWIZZLE_128B, two boxes per 128-wide MN panel 8192 B
// apart (MN-major: LBO 8192, SBO 1024, 16-row k-step 2048 B; scripts/probe_tf32.cu (e)).
struct EncMaps {
    CUtensorMap hi[kMaxT], lo[kMaxT];
    int use;
};
bool encode_tmap_bf16_2d(CUtensorMap* m, const void* base, int64_t width, int64_t rows, int64_t ld, int box_w,
                         int box_h);

struct EnCursor {
    int64_t tile;      // >= total: exhausted
    int t, p, KP;
    int64_t row0, rlim;
    int m0, n0;
};

__device__ __forceinline__ int64_t type_rows(const HopMeta* m, int t) { return m->src_off[t + 1] - m->src_off[t]; }

// ---- forward tiles: (projected type t, 128-row block, 128-col block) -------------------
__device__ __forceinline__ int64_t fwd_total(const EncDev& e, const HopMeta* m, int nct) {
    int64_t tot = 0;
    for (int t = 0; t < e.T; ++t)
        if (e.proj[t]) tot += ((type_rows(m, t) + 127) / 128) * nct;
    return tot;
}
__device__ __forceinline__ void fwd_decode(const EncDev& e, const HopMeta* m, int nct, EnCursor& c) {
    int64_t rem = c.tile;
    for (int t = 0; t < e.T; ++t) {
        if (!e.proj[t]) continue;
        const int64_t nt = ((type_rows(m, t) + 127) / 128) * nct;
        if (rem < nt) {
            c.t = t;
            c.row0 = m->src_off[t] + (rem / nct) * 128;
            c.rlim = m->src_off[t + 1];
            c.n0 = (int)(rem % nct) * 128;
            c.m0 = 0;
            c.KP = e.dim[t] / 64;
            c.p = 0;
            return;
        }
        rem -= nt;
    }
}

// ---- weight-gradient items: (type t, row chunk, 128-row block of dW, 128-col block) ------
__device__ __forceinline__ int64_t dw_rpc(const EncDev& e, const HopMeta* m, int t, int nct, int grid) {
    const int64_t n = type_rows(m, t);
    const int64_t want = (n * (e.dim[t] / 128) * nct + 2 * grid - 1) / (2 * grid);   // ~2 items per CTA
    return max((int64_t)256, (want + 63) / 64 * 64);
}
__device__ __forceinline__ int64_t dw_total(const EncDev& e, const HopMeta* m, int nct, int grid) {
    int64_t tot = 0;
    for (int t = 0; t < e.T; ++t) {
        if (!e.proj[t]) continue;
        const int64_t rpc = dw_rpc(e, m, t, nct, grid);
        tot += ((type_rows(m, t) + rpc - 1) / rpc) * (e.dim[t] / 128) * nct;
    }
    return tot;
}
__device__ __forceinline__ void dw_decode(const EncDev& e, const HopMeta* m, int nct, int grid, EnCursor& c) {
    int64_t rem = c.tile;
    for (int t = 0; t < e.T; ++t) {
        if (!e.proj[t]) continue;
        const int64_t rpc = dw_rpc(e, m, t, nct, grid);
        const int mt = e.dim[t] / 128;
        const int64_t nt = ((type_rows(m, t) + rpc - 1) / rpc) * mt * nct;
        if (rem < nt) {
            c.t = t;
            const int64_t chunk = rem / (mt * nct);
            const int q = (int)(rem % (mt * nct));
            c.m0 = (q / nct) * 128;
            c.n0 = (q % nct) * 128;
            c.row0 = m->src_off[t] + chunk * rpc;
            c.rlim = min(m->src_off[t + 1], c.row0 + rpc);
            c.KP = (int)((c.rlim - c.row0 + 63) / 64);
            c.p = 0;
            return;
        }
        rem -= nt;
    }
}

// ---- the warp-specialized pipelined kernel (BWD = false: forward, true: weight gradient) --
// warps 0-3: A producers (cp.async gathers of the feature panels into a ring of EN_A_STAGES
//            stages; completion is signalled per stage with cp.async.mbarrier.arrive.noinc)
// warps 4-7: epilogue (TMEM -> registers -> H0 rows / red.add into dW), warp w drains TMEM
//            lanes 32*(w%4)..; two TMEM accumulators so a tile's epilogue overlaps the next
//            tile's MMAs
// warp 8:    lane 0 issues the tcgen05 MMAs and commits stage / accumulator barriers
// warp 9:    lane 0 is the B producer (TMA boxes of W^T / dH0 hi + lo into a ring of EN_B_STAGES)
constexpr int EN_WS_THREADS = 320;

__device__ __forceinline__ void cp_arrive_noinc(uint64_t* bar) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(umma::smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(umma::smem_u32(bar))
                 : "memory");
}

template <bool BWD>
__global__ void __launch_bounds__(EN_WS_THREADS, 1) enc_umma_kernel(GraphDev g, EncDev e, const HopMeta* __restrict__ m,
                                                                    const int64_t* __restrict__ src_gid,
                                                                    float* __restrict__ H0, EncOut out,
                                                                    const __grid_constant__ EncMaps maps) {
    GSB_PDL_ENTRY();
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int EN_A_STAGES = EnRing<BWD>::A, EN_B_STAGES = EnRing<BWD>::B;
    static_assert(EN_A_STAGES * EN_PANEL + EN_B_STAGES * EN_B_STAGE <= 192 * 1024, "encoder rings exceed 192 KB");
    __shared__ __align__(8) uint64_t fullA[EN_A_STAGES], emptyA[EN_A_STAGES], fullB[EN_B_STAGES], emptyB[EN_B_STAGES];
    __shared__ __align__(8) uint64_t tfull[2], tempty[2];
    __shared__ uint32_t tmem_sh;
    uint8_t* ringA = smem;
    uint8_t* ringB = smem + EN_A_STAGES * EN_PANEL;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (warp == 0) umma::tmem_alloc<256>(&tmem_sh);
    if (tid == 0) {
        for (int s = 0; s < EN_A_STAGES; ++s) {
            umma::mbar_init(&fullA[s], 128);
            umma::mbar_init(&emptyA[s], 1);
        }
        for (int s = 0; s < EN_B_STAGES; ++s) {
            umma::mbar_init(&fullB[s], 1);
            umma::mbar_init(&emptyB[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            umma::mbar_init(&tfull[a], 1);
            umma::mbar_init(&tempty[a], 128);
        }
        umma::fence_barrier_init();
    }
    umma::tc_fence_before();
    __syncthreads();
    umma::tc_fence_after();
    const uint32_t tmem = tmem_sh;
    const int nct = e.d_out / 128;
    const int grid = gridDim.x;
    const int64_t total = BWD ? dw_total(e, m, nct, grid) : fwd_total(e, m, nct);
    auto decode = [&](EnCursor& c) {
        if (BWD) dw_decode(e, m, nct, grid, c);
        else fwd_decode(e, m, nct, c);
    };

    if (warp < 4) {
        // ------------------------------------------------------------------ producers
        const int p = tid;                       // 0..127
        int64_t it = 0;
        for (int64_t tile = blockIdx.x; tile < total; tile += grid) {
            EnCursor c;
            c.tile = tile;
            decode(c);
            if (!BWD) {
                // rows rg + 16 i (i < 8), 16-B chunk ch of each 128-B K slice: a warp covers 4 whole rows
                const int ch = p & 7, rg = p >> 3;
                const char* arow[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int64_t row = c.row0 + rg + 16 * i;
                    arow[i] = row < c.rlim ? reinterpret_cast<const char*>(feat_row(g, __ldg(src_gid + row))) : nullptr;
                }
                const char* zsrc = reinterpret_cast<const char*>(e.wt_hi[c.t]);   // any valid address (0-byte copies)
                for (int pn = 0; pn < c.KP; ++pn, ++it) {
                    const int st = (int)(it % EN_A_STAGES);
                    if (it >= EN_A_STAGES) umma::mbar_wait(&emptyA[st], (uint32_t)((it / EN_A_STAGES) - 1) & 1u);
                    const uint32_t sA = umma::smem_u32(ringA + st * EN_PANEL);
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int r = rg + 16 * i;
                        const uint32_t o = umma::kmaj16_chunk(r, ch);
                        cp16(sA + o, arow[i] ? arow[i] + pn * 128 + ch * 16 : zsrc, arow[i] ? 16 : 0);
                    }
                    cp_arrive_noinc(&fullA[st]);
                }
            } else {
                // K rows kr = (p >> 4) + 8 i (i < 8) of the 64-row panel, 16-B chunk c of the 128-wide slice
                const int cc = p & 15, kb = p >> 4;
                int64_t gid_next[8];
                auto load_gids = [&](int pn) {
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int64_t row = c.row0 + (int64_t)pn * 64 + kb + 8 * i;
                        gid_next[i] = row < c.rlim ? __ldg(src_gid + row) : -1;
                    }
                };
                load_gids(0);
                for (int pn = 0; pn < c.KP; ++pn, ++it) {
                    int64_t gid[8];
#pragma unroll
                    for (int i = 0; i < 8; ++i) gid[i] = gid_next[i];
                    if (pn + 1 < c.KP) load_gids(pn + 1);       // prefetch the next panel's ids
                    const int st = (int)(it % EN_A_STAGES);
                    if (it >= EN_A_STAGES) umma::mbar_wait(&emptyA[st], (uint32_t)((it / EN_A_STAGES) - 1) & 1u);
                    const uint32_t sA = umma::smem_u32(ringA + st * EN_PANEL);
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int kr = kb + 8 * i;
                        const bool ok = gid[i] >= 0;
                        const uint32_t o = umma::mnmaj16_chunk(cc * 8, kr);
                        const char* src = ok ? reinterpret_cast<const char*>(feat_row(g, gid[i])) + (size_t)(c.m0 + cc * 8) * 2
                                             : reinterpret_cast<const char*>(e.d_hi);
                        cp16(sA + o, src, ok ? 16 : 0);
                    }
                    cp_arrive_noinc(&fullA[st]);
                }
            }
        }
    } else if (warp == 9) {
        if (lane == 0) {
            // -------------------------------------------------------------- B producer (TMA)
            int64_t it = 0;
            for (int64_t tile = blockIdx.x; tile < total; tile += grid) {
                EnCursor c;
                c.tile = tile;
                decode(c);
                for (int pn = 0; pn < c.KP; ++pn, ++it) {
                    const int sb = (int)(it % EN_B_STAGES);
                    if (it >= EN_B_STAGES) umma::mbar_wait(&emptyB[sb], (uint32_t)((it / EN_B_STAGES) - 1) & 1u);
                    const uint32_t bh = umma::smem_u32(ringB + sb * EN_B_STAGE), bl = bh + EN_PANEL;
                    tma::mbar_expect_tx(&fullB[sb], 2 * EN_PANEL);
                    if (!BWD) {            // W_t^T hi / lo panels: two TMA boxes {64, 128}
                        tma::load_2d(bh, &maps.hi[c.t], pn * 64, c.n0, &fullB[sb]);
                        tma::load_2d(bl, &maps.lo[c.t], pn * 64, c.n0, &fullB[sb]);
                    } else {               // dH0 hi / lo rows of this panel: 2 x 2 boxes {64, 64}
                        const int32_t r0 = (int32_t)(c.row0 + (int64_t)pn * 64);
                        tma::load_2d(bh, &maps.hi[0], c.n0, r0, &fullB[sb]);
                        tma::load_2d(bh + 8192, &maps.hi[0], c.n0 + 64, r0, &fullB[sb]);
                        tma::load_2d(bl, &maps.lo[0], c.n0, r0, &fullB[sb]);
                        tma::load_2d(bl + 8192, &maps.lo[0], c.n0 + 64, r0, &fullB[sb]);
                    }
                }
            }
        }
    } else if (warp == 8) {
        if (lane == 0) {
            // -------------------------------------------------------------- MMA issuer
            constexpr uint32_t IDESC = umma::idesc_bf16(128, BWD, BWD);
            int64_t it = 0, j = 0;
            for (int64_t tile = blockIdx.x; tile < total; tile += grid, ++j) {
                EnCursor c;
                c.tile = tile;
                decode(c);
                const int acc = (int)(j & 1);
                if (j >= 2) umma::mbar_wait(&tempty[acc], (uint32_t)((j >> 1) - 1) & 1u);
                umma::tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(acc * 128);
                for (int pn = 0; pn < c.KP; ++pn, ++it) {
                    const int st = (int)(it % EN_A_STAGES), sb = (int)(it % EN_B_STAGES);
                    umma::mbar_wait(&fullA[st], (uint32_t)(it / EN_A_STAGES) & 1u);
                    umma::mbar_wait(&fullB[sb], (uint32_t)(it / EN_B_STAGES) & 1u);
                    umma::fence_proxy_async_smem();
                    umma::tc_fence_after();
                    const uint32_t a = umma::smem_u32(ringA + st * EN_PANEL);
                    const uint32_t bh = umma::smem_u32(ringB + sb * EN_B_STAGE), bl = bh + EN_PANEL;
#pragma unroll
                    for (int ks = 0; ks < 4; ++ks) {
                        const uint32_t o = BWD ? ks * 4096u : ks * 32u;
                        const uint64_t da = BWD ? umma::desc_mnmajor16(a + o) : umma::desc_kmajor(a + o);
                        // backward B from TMA boxes: MN atoms 8192 B apart, 8-row K groups 1024 B, k-step 2048 B
                        const uint64_t dbh = !BWD ? umma::desc_kmajor(bh + o) : umma::desc_encode(bh + ks * 2048u, 8192, 1024, 2);
                        const uint64_t dbl = !BWD ? umma::desc_kmajor(bl + o) : umma::desc_encode(bl + ks * 2048u, 8192, 1024, 2);
                        umma::mma_f16(d, da, dbh, IDESC, (pn > 0 || ks > 0) ? 1u : 0u);
                        umma::mma_f16(d, da, dbl, IDESC, 1u);
                    }
                    umma::mma_commit(&emptyA[st]);
                    umma::mma_commit(&emptyB[sb]);
                }
                umma::mma_commit(&tfull[acc]);
            }
        }
    } else {
        // ------------------------------------------------------------------ epilogue (warps 4-7)
        static_assert(EN_WS_THREADS == 320, "warp roles: 0-3 A producers, 4-7 epilogue, 8 MMA, 9 B producer");
        const int q = warp & 3;
        const int r = q * 32 + lane;
        int64_t j = 0;
        for (int64_t tile = blockIdx.x; tile < total; tile += grid, ++j) {
            EnCursor c;
            c.tile = tile;
            decode(c);
            const int acc = (int)(j & 1);
            umma::mbar_wait(&tfull[acc], (uint32_t)(j >> 1) & 1u);
            umma::tc_fence_after();
#pragma unroll 1
            for (int cc = 0; cc < 4; ++cc) {
                float v[32];
                umma::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * 128 + cc * 32), v);
                if (!BWD) {
                    const int64_t row = c.row0 + r;
                    if (row < c.rlim) {
                        float4* o4 = reinterpret_cast<float4*>(H0 + row * e.d_out + c.n0 + cc * 32);
#pragma unroll
                        for (int k = 0; k < 8; ++k) o4[k] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
                    }
                } else {   // dW_t[m0 + r][n0 + ..] += D (row chunks of other CTAs add in)
                    float* o = out.dW[c.t] + (int64_t)(c.m0 + r) * e.d_out + c.n0 + cc * 32;
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        red_add_f4(o + 4 * k, make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]));
                }
            }
            umma::tc_fence_before();
            mbar_arrive(&tempty[acc]);
        }
    }
    __syncthreads();
    if (warp == 0) {
        umma::tc_fence_after();
        umma::tmem_dealloc<256>(tmem);
    }
}

}  // namespace gsb

namespace gsb {

// W_t [dim][d_out] fp32 -> transposed bf16 hi / lo [d_out][dim]
__global__ void enc_wsplit_kernel(const float* __restrict__ W, int dim, int d_out, __nv_bfloat16* __restrict__ hi,
                                  __nv_bfloat16* __restrict__ lo) {
    GSB_PDL_ENTRY();
    const int64_t n = (int64_t)dim * d_out;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int k = (int)(i / d_out), j = (int)(i % d_out);
        const float x = W[i];
        const __nv_bfloat16 h = __float2bfloat16_rn(x);
        hi[(int64_t)j * dim + k] = h;
        lo[(int64_t)j * dim + k] = __float2bfloat16_rn(x - __bfloat162float(h));
    }
}

// dH0 rows of projected types -> bf16 hi / lo (same layout [rows][d_out])
__global__ void enc_dsplit_kernel(EncDev e, const HopMeta* __restrict__ m, const float* __restrict__ dH0,
                                  __nv_bfloat16* __restrict__ hi, __nv_bfloat16* __restrict__ lo) {
    GSB_PDL_ENTRY();
    const int64_t n4 = m->n_src * (int64_t)e.d_out / 4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i * 4 / e.d_out;
        int t = 0;
        for (int k = 1; k < e.T; ++k) t += (row >= m->src_off[k]) ? 1 : 0;
        if (!e.proj[t]) continue;
        const float4 x = reinterpret_cast<const float4*>(dH0)[i];
        const float xs[4] = {x.x, x.y, x.z, x.w};
        __nv_bfloat16 h[4], l[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            h[u] = __float2bfloat16_rn(xs[u]);
            l[u] = __float2bfloat16_rn(xs[u] - __bfloat162float(h[u]));
        }
        reinterpret_cast<uint2*>(hi)[i] = *reinterpret_cast<const uint2*>(h);
        reinterpret_cast<uint2*>(lo)[i] = *reinterpret_cast<const uint2*>(l);
    }
}

// frozen-table rows (non-projected ntypes): H0[row] = widen(F_t[local]), one 16-B chunk per thread
template <bool BF16>
__global__ void enc_copy_kernel(GraphDev g, EncDev e, const HopMeta* __restrict__ m, const int64_t* __restrict__ src_gid,
                                float* __restrict__ H0) {
    GSB_PDL_ENTRY();
    constexpr int V = Chunk<BF16>::kVec;
    const int cpr = e.d_out / V;                        // chunks per row (dim_t == d_out)
    const int64_t n = m->n_src * (int64_t)cpr;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i / cpr;
        const int c = (int)(i - row * cpr);
        int t = 0;
        for (int k = 1; k < e.T; ++k) t += (row >= m->src_off[k]) ? 1 : 0;
        if (e.proj[t]) continue;
        float r[V];
#pragma unroll
        for (int v = 0; v < V; ++v) r[v] = 0.f;
        chunk_acc<BF16>(r, ldg_nc_u4(feat_row(g, __ldg(src_gid + row)) + c));
        float4* o4 = reinterpret_cast<float4*>(H0 + row * e.d_out + (int64_t)c * V);
#pragma unroll
        for (int v = 0; v < V; v += 4) o4[v / 4] = make_float4(r[v], r[v + 1], r[v + 2], r[v + 3]);
    }
}

// workspace layout: per projected ntype wt_hi, wt_lo [d_out][dim_t] bf16; then d_hi, d_lo
// [cap_rows][d_out] bf16 (each piece 256-B aligned)
static size_t enc_layout(const Graph* G, const float* const* W, int d_out, int64_t cap_rows, EncDev* e,
                         char* base) {
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off = align_up(off + bytes);
        return base ? base + o : nullptr;
    };
    if (e) {
        memset(e, 0, sizeof(EncDev));
        e->T = G->dev.T;
        e->d_out = d_out;
    }
    for (int t = 0; t < G->dev.T; ++t) {
        if (!W[t]) continue;
        const size_t b = (size_t)d_out * G->dev.dim_t[t] * 2;
        char* h = take(b);
        char* l = take(b);
        if (e) {
            e->proj[t] = 1;
            e->wt_hi[t] = reinterpret_cast<const __nv_bfloat16*>(h);
            e->wt_lo[t] = reinterpret_cast<const __nv_bfloat16*>(l);
        }
    }
    for (int t = 0; e && t < G->dev.T; ++t) e->dim[t] = G->dev.dim_t[t];
    char* dh = take((size_t)cap_rows * d_out * 2);
    char* dl = take((size_t)cap_rows * d_out * 2);
    if (e) {
        e->d_hi = reinterpret_cast<const __nv_bfloat16*>(dh);
        e->d_lo = reinterpret_cast<const __nv_bfloat16*>(dl);
    }
    return off;
}

static gsb_status enc_check(const Blocks* B, const float* const* W, int d_out) {
    const Graph* G = B->g;
    GSB_CHECK_ARG(W, "null W_in array");
    GSB_CHECK_ARG(d_out > 0 && d_out % 128 == 0, "d_out %d must be a multiple of 128", d_out);
    for (int t = 0; t < G->dev.T; ++t) {
        GSB_CHECK_ARG(G->dev.feat[t], "features of ntype %d not registered", t);
        if (W[t]) {
            GSB_CHECK_ARG(G->dev.feat_dtype == GSB_BF16, "projected ntypes need bf16 feature rows");
            GSB_CHECK_ARG(G->dev.dim_t[t] % 128 == 0, "projected ntype %d: width %d not a multiple of 128", t,
                          G->dev.dim_t[t]);
        } else {
            GSB_CHECK_ARG(G->dev.dim_t[t] == d_out, "frozen ntype %d: width %d != d_out %d", t, G->dev.dim_t[t], d_out);
        }
    }
    return GSB_OK;
}

// B operand by TMA (the kernel has no other B path: a map that cannot be encoded is an error)
template <bool BWD>
static gsb_status launch_enc(const char* name, const GraphDev& g, const EncDev& e, const HopMeta* m,
                             const int64_t* src_gid, float* H0, const EncOut& out, int64_t cap_rows, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        GSB_CUDA(cudaFuncSetAttribute(enc_umma_kernel<BWD>, cudaFuncAttributeMaxDynamicSharedMemorySize, EN_SMEM));
        attr = true;
    }
    EncMaps maps;
    memset(&maps, 0, sizeof(maps));
    bool ok = true;
    if (ok && !BWD) {
        for (int t = 0; t < e.T && ok; ++t)
            if (e.proj[t])
                ok = encode_tmap_bf16_2d(&maps.hi[t], e.wt_hi[t], e.dim[t], e.d_out, e.dim[t], 64, 128) &&
                     encode_tmap_bf16_2d(&maps.lo[t], e.wt_lo[t], e.dim[t], e.d_out, e.dim[t], 64, 128);
    } else if (ok) {
        ok = encode_tmap_bf16_2d(&maps.hi[0], e.d_hi, e.d_out, cap_rows, e.d_out, 64, 64) &&
             encode_tmap_bf16_2d(&maps.lo[0], e.d_lo, e.d_out, cap_rows, e.d_out, 64, 64);
    }
    GSB_CHECK_ARG(ok, "%s: TMA descriptors of the B operand could not be encoded", name);
    maps.use = 1;
    GSB_LAUNCH(name, enc_umma_kernel<BWD>, kNumSMs, EN_WS_THREADS, EN_SMEM, s, g, e, m, src_gid, H0, out, maps);
    return GSB_OK;
}

}  // namespace gsb

using namespace gsb;

extern "C" {

gsb_status gsb_encoder_ws_bytes(gsb_blocks_t b, const float* const* W_in, int32_t d_out, size_t* bytes) {
    Blocks* B = reinterpret_cast<Blocks*>(b);
    GSB_CHECK_ARG(B && W_in && bytes, "null argument");
    *bytes = enc_layout(B->g, W_in, d_out, B->cap_dst[B->L + 1], nullptr, nullptr);
    return GSB_OK;
}

gsb_status gsb_encoder_fwd(gsb_blocks_t b, const void* arena, const float* const* W_in, int32_t d_out, float* H0,
                           void* ws, size_t ws_bytes, void* stream) {
    Blocks* B = reinterpret_cast<Blocks*>(b);
    GSB_CHECK_ARG(B && arena && H0 && ws, "null argument");
    gsb_status st = enc_check(B, W_in, d_out);
    if (st != GSB_OK) return st;
    EncDev e;
    const size_t need = enc_layout(B->g, W_in, d_out, B->cap_dst[B->L + 1], &e, static_cast<char*>(ws));
    GSB_CHECK_ARG(ws_bytes >= need, "workspace %zu < %zu bytes", ws_bytes, need);
    cudaStream_t s = (cudaStream_t)stream;
    const GraphDev& g = B->g->dev;
    HopBufs hb = B->hop(B->L, const_cast<void*>(arena));
    bool any_proj = false, any_frozen = false;
    for (int t = 0; t < g.T; ++t) {
        if (!W_in[t]) {
            any_frozen = true;
            continue;
        }
        any_proj = true;
        GSB_LAUNCH("enc_wsplit", enc_wsplit_kernel, grid_for((int64_t)g.dim_t[t] * d_out, 256), 256, 0, s, W_in[t],
                   g.dim_t[t], d_out, const_cast<__nv_bfloat16*>(e.wt_hi[t]), const_cast<__nv_bfloat16*>(e.wt_lo[t]));
    }
    if (any_frozen) {
        const int grid = grid_for(hb.cap_src * (d_out / 8), 256, kNumSMs * 8);
        if (g.feat_dtype == GSB_BF16) {
            GSB_LAUNCH("enc_copy", enc_copy_kernel<true>, grid, 256, 0, s, g, e, hb.meta, hb.src_gid, H0);
        } else {
            GSB_LAUNCH("enc_copy", enc_copy_kernel<false>, grid, 256, 0, s, g, e, hb.meta, hb.src_gid, H0);
        }
    }
    if (any_proj) {
        EncOut out{};
        return launch_enc<false>("enc_gemm_fwd", g, e, hb.meta, hb.src_gid, H0, out, B->cap_dst[B->L + 1], s);
    }
    return GSB_OK;
}

gsb_status gsb_encoder_bwd(gsb_blocks_t b, const void* arena, const float* const* W_in, const float* dH0, int32_t d_out,
                           float* const* dW_in, void* ws, size_t ws_bytes, void* stream) {
    Blocks* B = reinterpret_cast<Blocks*>(b);
    GSB_CHECK_ARG(B && arena && dH0 && dW_in && ws, "null argument");
    gsb_status st = enc_check(B, W_in, d_out);
    if (st != GSB_OK) return st;
    EncDev e;
    const size_t need = enc_layout(B->g, W_in, d_out, B->cap_dst[B->L + 1], &e, static_cast<char*>(ws));
    GSB_CHECK_ARG(ws_bytes >= need, "workspace %zu < %zu bytes", ws_bytes, need);
    cudaStream_t s = (cudaStream_t)stream;
    const GraphDev& g = B->g->dev;
    HopBufs hb = B->hop(B->L, const_cast<void*>(arena));
    EncOut out{};
    bool any = false;
    for (int t = 0; t < g.T; ++t) {
        if (!W_in[t]) continue;
        GSB_CHECK_ARG(dW_in[t], "dW_in[%d] missing for a projected ntype", t);
        out.dW[t] = dW_in[t];
        GSB_CUDA(cudaMemsetAsync(dW_in[t], 0, sizeof(float) * (size_t)g.dim_t[t] * d_out, s));
        any = true;
    }
    if (!any) return GSB_OK;
    GSB_LAUNCH("enc_dsplit", enc_dsplit_kernel, grid_for(hb.cap_src * d_out / 4, 256, kNumSMs * 8), 256, 0, s, e,
               hb.meta, dH0, const_cast<__nv_bfloat16*>(e.d_hi), const_cast<__nv_bfloat16*>(e.d_lo));
    return launch_enc<true>("enc_gemm_dW", g, e, hb.meta, hb.src_gid, nullptr, out, B->cap_dst[B->L + 1], s);
}

}  // extern "C"
