// gemm_simt.cuh -- the grouped RGCN GEMMs (modes NN / NT / TN of gemm_umma.cuh, same UProb
// problem statement) for SMALL problems: plain fp32 FMA on 32 x 32 output tiles, 64 threads
// per tile (4 x 4 outputs per thread), K in 32-wide chunks staged through double-buffered
// shared memory, split-K / row chunks over many CTAs.
//
// Why: at the top layer and the decoder the GEMMs are 1024 rows x 128..640 (tens of MFLOP).
// A tcgen05 tile pipeline spends ~10 us there on its fixed costs (TMEM alloc, barrier init,
// the first TMA round trip, one 128 x 128 tile epilogue, a 225 KB CTA that waits for a whole
// SM), while the math is ~1 us of FMA spread over 148 SMs; here hundreds of small CTAs start at
// once and share SMs with the concurrently running sample phase.  fp32 FMA accumulation keeps
// the result within the north_star 1e-5 tolerance (better than 3xTF32).
#pragma once
#include "gemm_umma.cuh"

namespace gsb {

constexpr int SG_T = 32;        // output tile (rows x cols) and K chunk
constexpr int SG_THREADS = 64;  // 8 x 8 threads, 4 x 4 outputs each
constexpr int SG_LD = SG_T + 4; // smem row stride (floats), keeps float4 reads aligned

// tile counts of group t.  NN: row tiles x col tiles x ksplit (K = slots * d_in).  NT: row tiles
// x (slots x d_in tiles) x ksplit (K = N).  TN: (slots x d_in tiles) x col tiles x row chunks.
template <int MODE>
__device__ __forceinline__ int64_t sg_tiles_of_group(const UProb& P, int t, int64_t rows) {
    const int64_t rt = (rows + SG_T - 1) / SG_T;
    const int ct = (P.N + SG_T - 1) / SG_T, kt = (P.d_in + SG_T - 1) / SG_T;
    if (MODE == UMMA_NN) return rt * ct * P.ksplit;
    if (MODE == UMMA_NT) return rt * P.rg.ks[t] * kt * P.ksplit;
    return (int64_t)P.rg.ks[t] * kt * ct * ((rows + P.rows_per_chunk - 1) / P.rows_per_chunk);
}

template <int MODE>
__global__ void __launch_bounds__(SG_THREADS) simt_gemm_kernel(UProb P) {
    GSB_PDL_ENTRY();
    __shared__ __align__(16) float As[2][SG_T][SG_LD];   // [k][m]
    __shared__ __align__(16) float Bs[2][SG_T][SG_LD];   // [k][n]
    const int tid = threadIdx.x;
    // ---- decode this CTA's tile
    int64_t rem = blockIdx.x;
    int t = 0;
    int64_t r0 = 0, r1 = 0;
    for (;; ++t) {
        if (t >= P.rg.G) return;
        group_rows(P.rg, t, r0, r1);
        const int64_t nt = sg_tiles_of_group<MODE>(P, t, r1 - r0);
        if (rem < nt) break;
        rem -= nt;
    }
    const int ct = (P.N + SG_T - 1) / SG_T, kt = (P.d_in + SG_T - 1) / SG_T;
    int64_t row0 = 0, rlim = 0;
    int s = 0, c0 = 0, n0 = 0, split = 0, p0 = 0, p1 = 0;
    if (MODE == UMMA_NN) {
        split = (int)(rem % P.ksplit); rem /= P.ksplit;
        n0 = (int)(rem % ct) * SG_T; rem /= ct;
        row0 = r0 + rem * SG_T; rlim = r1;
        const int kp = P.rg.ks[t] * kt;                   // K chunks: slot-major, d_in / 32 each
        p0 = (int)((int64_t)split * kp / P.ksplit); p1 = (int)((int64_t)(split + 1) * kp / P.ksplit);
    } else if (MODE == UMMA_NT) {
        split = (int)(rem % P.ksplit); rem /= P.ksplit;
        const int q = (int)(rem % (P.rg.ks[t] * kt)); rem /= (P.rg.ks[t] * kt);
        s = q / kt; c0 = (q % kt) * SG_T;
        row0 = r0 + rem * SG_T; rlim = r1;
        const int kp = (P.N + SG_T - 1) / SG_T;
        p0 = (int)((int64_t)split * kp / P.ksplit); p1 = (int)((int64_t)(split + 1) * kp / P.ksplit);
    } else {
        n0 = (int)(rem % ct) * SG_T; rem /= ct;
        const int q = (int)(rem % (P.rg.ks[t] * kt)); rem /= (P.rg.ks[t] * kt);
        s = q / kt; c0 = (q % kt) * SG_T;
        row0 = r0 + rem * P.rows_per_chunk;
        rlim = min(r1, row0 + (int64_t)P.rows_per_chunk);
        p0 = 0; p1 = (int)((rlim - row0 + SG_T - 1) / SG_T);
    }
    // ---- chunk loads: thread covers line tid/2 of the chunk, 16 consecutive elements
    const int li = tid >> 1, lo = (tid & 1) * 16;
    float ra[16], rb[16];
    auto load = [&](int p) {
        if (MODE == UMMA_NN) {
            const int sp = p / kt, kk = (p - sp * kt) * SG_T;
            const int64_t row = row0 + li;
            const float* a = P.A + row * P.lda + (int64_t)sp * P.d_in + kk + lo;
#pragma unroll
            for (int i = 0; i < 16; ++i) ra[i] = (row < rlim && kk + lo + i < P.d_in) ? __ldg(a + i) : 0.f;
            const float* w = P.B + (int64_t)P.rg.slot_w[t][sp] * P.bslot + (int64_t)(kk + li) * P.ldb + n0 + lo;
#pragma unroll
            for (int i = 0; i < 16; ++i) rb[i] = (kk + li < P.d_in && n0 + lo + i < P.N) ? __ldg(w + i) : 0.f;
        } else if (MODE == UMMA_NT) {
            const int nn = p * SG_T;
            const int64_t row = row0 + li;
            const float* a = P.A + row * P.lda + nn + lo;
#pragma unroll
            for (int i = 0; i < 16; ++i) ra[i] = (row < rlim && nn + lo + i < P.N) ? __ldg(a + i) : 0.f;
            const float* w = P.B + (int64_t)P.rg.slot_w[t][s] * P.bslot + (int64_t)(c0 + li) * P.ldb + nn + lo;
#pragma unroll
            for (int i = 0; i < 16; ++i) rb[i] = (c0 + li < P.d_in && nn + lo + i < P.N) ? __ldg(w + i) : 0.f;
        } else {
            const int64_t row = row0 + (int64_t)p * SG_T + li;
            const float* a = P.A + row * P.lda + (int64_t)s * P.d_in + c0 + lo;
#pragma unroll
            for (int i = 0; i < 16; ++i) ra[i] = (row < rlim && c0 + lo + i < P.d_in) ? __ldg(a + i) : 0.f;
            const float* b = P.B + row * P.ldb + n0 + lo;
#pragma unroll
            for (int i = 0; i < 16; ++i) rb[i] = (row < rlim && n0 + lo + i < P.N) ? __ldg(b + i) : 0.f;
        }
    };
    // NN / NT chunks hold A as [m][k] and are transposed into As[k][m]; NT's B is W[kk][n] ->
    // Bs[n][kk]; TN's chunks are already [k = row][m] and [k = row][n]
    auto store = [&](int buf) {
        if (MODE == UMMA_TN) {
#pragma unroll
            for (int i = 0; i < 16; ++i) As[buf][li][lo + i] = ra[i];
        } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) As[buf][lo + i][li] = ra[i];
        }
        if (MODE == UMMA_NT) {
#pragma unroll
            for (int i = 0; i < 16; ++i) Bs[buf][lo + i][li] = rb[i];
        } else {
#pragma unroll
            for (int i = 0; i < 16; ++i) Bs[buf][li][lo + i] = rb[i];
        }
    };
    const int tx = tid & 7, ty = tid >> 3;      // outputs: rows ty*4.., cols tx*4..
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
    // TN bias gradient: column sums of dZ over the chunk rows (last slot, first k tile)
    const bool do_db = (MODE == UMMA_TN) && P.db && s == P.rg.ks[t] - 1 && c0 == 0;
    float dbs = 0.f;
    if (p0 < p1) {
        load(p0);
        store(0);
        __syncthreads();
        for (int p = p0; p < p1; ++p) {
            const int buf = (p - p0) & 1;
            if (p + 1 < p1) load(p + 1);          // next chunk in flight during this one's FMAs
#pragma unroll
            for (int k = 0; k < SG_T; ++k) {
                const float4 a = *reinterpret_cast<const float4*>(&As[buf][k][ty * 4]);
                const float4 b = *reinterpret_cast<const float4*>(&Bs[buf][k][tx * 4]);
                const float av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
                for (int i = 0; i < 4; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
            }
            if (do_db && tid < SG_T) {
#pragma unroll 8
                for (int k = 0; k < SG_T; ++k) dbs += Bs[buf][k][tid];
            }
            if (p + 1 < p1) store(buf ^ 1);
            __syncthreads();
        }
    }
    // ---- epilogue
    if (MODE == UMMA_NN) {
        const bool split_k = P.ksplit > 1;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t row = row0 + ty * 4 + i;
            if (row >= rlim) continue;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int n = n0 + tx * 4 + j;
                if (n >= P.N) continue;
                float x = acc[i][j] + ((P.bias && split == 0) ? __ldg(P.bias + n) : 0.f);
                float* o = P.C + row * P.ldc + n;
                if (split_k) atomicAdd(o, x);
                else *o = P.relu ? fmaxf(x, 0.f) : x;
            }
        }
    } else if (MODE == UMMA_NT) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int64_t row = row0 + ty * 4 + i;
            if (row >= rlim) continue;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int k = c0 + tx * 4 + j;
                if (k >= P.d_in) continue;
                float* o = P.C + row * P.ldc + (int64_t)s * P.d_in + k;
                if (P.ksplit > 1) atomicAdd(o, acc[i][j]);
                else *o = acc[i][j];
            }
        }
    } else {
        float* W = P.C + (int64_t)P.rg.slot_w[t][s] * P.bslot;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int k = c0 + ty * 4 + i;
            if (k >= P.d_in) continue;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int n = n0 + tx * 4 + j;
                if (n < P.N) atomicAdd(W + (int64_t)k * P.ldc + n, acc[i][j]);
            }
        }
        if (do_db && tid < SG_T && n0 + tid < P.N) atomicAdd(P.db + n0 + tid, dbs);
    }
}

// Launch when the problem is small (host-known row capacity <= SG_MAX_ROWS): returns false
// (nothing launched) otherwise.  NN / NT split K over CTAs unless relu is fused (caller's
// split-K contract: C zeroed first, no relu, bias from split 0).
constexpr int64_t SG_MAX_ROWS = 4096;
template <int MODE>
inline gsb_status launch_simt_gemm(const char* name, UProb P, int64_t rows_cap, cudaStream_t s, bool* launched) {
    *launched = false;
    if (rows_cap > SG_MAX_ROWS) return GSB_OK;
    const int ct = (P.N + SG_T - 1) / SG_T, kt = (P.d_in + SG_T - 1) / SG_T;
    int64_t rows_total = 0, base = 0;
    int max_ks = 1;
    for (int t = 0; t < P.rg.G; ++t) max_ks = std::max(max_ks, (int)P.rg.ks[t]);
    // host upper bound of the tiles: row capacity spread over the groups (+1 tile per group)
    rows_total = rows_cap + (int64_t)P.rg.G * SG_T;
    const int64_t rt = (rows_total + SG_T - 1) / SG_T;
    const int target = kNumSMs * 4;
    // split K only where the caller set up a split (C zeroed, no relu); any split count then works
    if (MODE == UMMA_NN) {
        base = rt * ct;
        const int kp = max_ks * kt;
        P.ksplit = (P.ksplit > 1 && base < target)
                       ? (int)std::max<int64_t>(1, std::min<int64_t>((target + base - 1) / base, std::max(1, kp / 2)))
                       : 1;
    } else if (MODE == UMMA_NT) {
        base = rt * max_ks * kt;
        const int kp = (P.N + SG_T - 1) / SG_T;
        P.ksplit = (P.ksplit > 1 && base < target)
                       ? (int)std::max<int64_t>(1, std::min<int64_t>((target + base - 1) / base, std::max(1, kp / 2)))
                       : 1;
    } else {
        // row chunks of a multiple of 32 rows sized for ~target CTAs
        const int64_t per = (int64_t)max_ks * kt * ct;
        int64_t rpc = (rows_total * per + target - 1) / target;
        rpc = std::max<int64_t>(64, (rpc + SG_T - 1) / SG_T * SG_T);
        P.rows_per_chunk = (int)rpc;
        base = per * ((rows_total + rpc - 1) / rpc + P.rg.G);
    }
    const int64_t tiles = (MODE == UMMA_TN) ? base : base * P.ksplit;
    *launched = true;
    GSB_LAUNCH(name, simt_gemm_kernel<MODE>, (int)std::max<int64_t>(1, tiles), SG_THREADS, 0, s, P);
    return GSB_OK;
}

}  // namespace gsb
