// gemm_umma.cuh -- grouped RGCN GEMMs on the 5th-gen tensor cores (tcgen05, TMEM).
//
// 3xTF32: every fp32 operand x is split into hi = rna_tf32(x), lo = rna_tf32(x - hi) while it
// is staged to shared memory, and D += A_hi B_hi + A_hi B_lo + A_lo B_hi is accumulated in
// TMEM (fp32).  The dropped lo*lo term and the tf32 rounding of lo keep the relative error
// near 2^-21 per product -- fp32-class, as the 1e-5 parity bar requires.
//
// Modes (same tile machinery, different operand index maps):
//   NN : C[r, n]          = act( sum_s A[r, s*d_in + k] W[slot_s][k][n] + bias[n] )   A K-major, B MN-major
//   NT : C[r, s*d_in + k] = sum_n dZ[r, n] W[slot_s][k][n]                          A K-major, B K-major
//   TN : dW[slot_s][k][n] += sum_{r in chunk} A[r, s*d_in + k] dZ[r, n]  (+ db)     A MN-major, B MN-major
// dZ = dH * 1[H > 0] when relu is set.  One CTA = 256 threads: all stage operands
// (global -> split -> st.shared, double-buffered), thread 0 issues the MMAs, all 8 warps
// drain the 128x128 fp32 accumulator from TMEM.  Persistent over tiles.
#pragma once
#include "gemm_simt.cuh"   // RowGroups
#include "gsb_internal.cuh"
#include "umma.cuh"

namespace gsb {

enum { UMMA_NN = 0, UMMA_NT = 1, UMMA_TN = 2 };

struct UProb {
    RowGroups rg;
    const float* A;        // NN: Acat/h ; NT: dH ; TN: Acat/h
    int64_t lda;
    const float* B;        // NN/NT: W ; TN: dH
    int64_t ldb;
    int64_t bslot;         // W slot stride (elements); 0 for a single matrix
    const float* H;        // relu mask source for dZ (NT: with A, TN: with B), may be null
    int relu;
    int d_in;              // K per slot (NN), output cols per slot (NT), output rows per slot (TN)
    int N;                 // output cols (NN, TN) / reduction length (NT)
    float* C;              // NN/NT output ; TN: dW
    int64_t ldc;
    const float* bias;     // NN
    float* db;             // TN (optional)
    int rows_per_chunk;    // TN
};

constexpr int UM_THREADS = 256;
constexpr int UM_PANEL = 16384;            // bytes of one 128 x 32 fp32/tf32 panel
constexpr int UM_STAGE = 4 * UM_PANEL;     // A_hi, A_lo, B_hi, B_lo
constexpr int UM_STAGES = 2;
constexpr int UM_SMEM = UM_STAGES * UM_STAGE + 1024;

__device__ __forceinline__ float4 ld4(const float* p, bool vec) {
    if (vec) return __ldg(reinterpret_cast<const float4*>(p));
    return make_float4(__ldg(p), __ldg(p + 1), __ldg(p + 2), __ldg(p + 3));
}

__device__ __forceinline__ void st_split(uint8_t* hi, uint8_t* lo, uint32_t off, float4 v) {
    uint32_t h0, h1, h2, h3, l0, l1, l2, l3;
    umma::split_tf32(v.x, h0, l0);
    umma::split_tf32(v.y, h1, l1);
    umma::split_tf32(v.z, h2, l2);
    umma::split_tf32(v.w, h3, l3);
    *reinterpret_cast<uint4*>(hi + off) = make_uint4(h0, h1, h2, h3);
    *reinterpret_cast<uint4*>(lo + off) = make_uint4(l0, l1, l2, l3);
}

// masked load of 4 consecutive elements [c, c+4) of row `row` (cols >= ncols -> 0)
__device__ __forceinline__ float4 load4(const float* base, int64_t ld, int64_t row, int64_t c, int64_t ncols, bool vec,
                                        const float* mask) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (c + 3 < ncols) {
        v = ld4(base + row * ld + c, vec);
        if (mask) {
            float4 h = ld4(mask + row * ld + c, vec);
            v.x = h.x > 0.f ? v.x : 0.f; v.y = h.y > 0.f ? v.y : 0.f;
            v.z = h.z > 0.f ? v.z : 0.f; v.w = h.w > 0.f ? v.w : 0.f;
        }
    } else if (c < ncols) {
        float e[4] = {0.f, 0.f, 0.f, 0.f};
        for (int q = 0; q < 4 && c + q < ncols; ++q) {
            float x = __ldg(base + row * ld + c + q);
            if (mask && __ldg(mask + row * ld + c + q) <= 0.f) x = 0.f;
            e[q] = x;
        }
        v = make_float4(e[0], e[1], e[2], e[3]);
    }
    return v;
}

template <int MODE>
__global__ void __launch_bounds__(UM_THREADS, 1) umma_gemm_kernel(UProb P) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    __shared__ __align__(8) uint64_t bars[UM_STAGES];
    __shared__ uint32_t tmem_sh;
    __shared__ float dbred[128];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const RowGroups& rg = P.rg;

    if (warp == 0) umma::tmem_alloc<128>(&tmem_sh);
    if (tid == 0) {
        for (int s = 0; s < UM_STAGES; ++s) umma::mbar_init(&bars[s], 1);
        umma::fence_barrier_init();
    }
    umma::tc_fence_before();
    __syncthreads();
    umma::tc_fence_after();
    const uint32_t tmem = tmem_sh;

    constexpr bool A_MN = (MODE == UMMA_TN);
    constexpr bool B_MN = (MODE != UMMA_NT);
    constexpr uint32_t IDESC = umma::idesc_tf32(128, A_MN, B_MN);
    const bool vecA = ((P.lda & 3) == 0) && ((reinterpret_cast<uintptr_t>(P.A) & 15) == 0);
    const bool vecB = ((P.ldb & 3) == 0) && ((reinterpret_cast<uintptr_t>(P.B) & 15) == 0);

    // ---- tile enumeration
    const int nct = (P.N + 127) / 128;          // NN/TN: output col tiles over N
    const int kct = (P.d_in + 127) / 128;       // NT: col tiles per slot; TN: row tiles over d_in
    int64_t total = 0;
    for (int t = 0; t < rg.G; ++t) {
        int64_t r0, r1;
        group_rows(rg, t, r0, r1);
        if (MODE == UMMA_NN) total += ((r1 - r0 + 127) / 128) * nct;
        else if (MODE == UMMA_NT) total += ((r1 - r0 + 127) / 128) * kct * rg.ks[t];
        else total += ((r1 - r0 + P.rows_per_chunk - 1) / P.rows_per_chunk) * rg.ks[t] * kct * nct;
    }

    uint32_t phase[UM_STAGES] = {0, 0};
    bool pend[UM_STAGES] = {false, false};
    int64_t it = 0;

    for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
        // ---- decode
        int t = 0;
        int64_t rem = tile, r0 = 0, r1 = 0;
        for (;; ++t) {
            group_rows(rg, t, r0, r1);
            int64_t nt;
            if (MODE == UMMA_NN) nt = ((r1 - r0 + 127) / 128) * nct;
            else if (MODE == UMMA_NT) nt = ((r1 - r0 + 127) / 128) * kct * rg.ks[t];
            else nt = ((r1 - r0 + P.rows_per_chunk - 1) / P.rows_per_chunk) * rg.ks[t] * kct * nct;
            if (rem < nt) break;
            rem -= nt;
        }
        int64_t row0 = 0, rlim = 0;   // NN/NT: output rows [row0, rlim); TN: reduction rows
        int s = 0, c0 = 0, n0 = 0, KP = 0;
        if (MODE == UMMA_NN) {
            row0 = r0 + (rem / nct) * 128;
            rlim = r1;
            n0 = (int)(rem % nct) * 128;
            KP = rg.ks[t] * (P.d_in / 32);
        } else if (MODE == UMMA_NT) {
            const int per = kct * rg.ks[t];
            row0 = r0 + (rem / per) * 128;
            rlim = r1;
            const int q = (int)(rem % per);
            s = q / kct;
            c0 = (q % kct) * 128;
            KP = (P.N + 31) / 32;
        } else {
            const int per = rg.ks[t] * kct * nct;
            row0 = r0 + (rem / per) * P.rows_per_chunk;
            rlim = min(r1, row0 + (int64_t)P.rows_per_chunk);
            int q = (int)(rem % per);
            s = q / (kct * nct);
            q -= s * kct * nct;
            c0 = (q / nct) * 128;   // k offset inside the slot
            n0 = (q % nct) * 128;
            KP = (int)((rlim - row0 + 31) / 32);
        }
        const bool do_db = (MODE == UMMA_TN) && P.db && (s == rg.ks[t] - 1) && c0 == 0;
        float4 cs = make_float4(0.f, 0.f, 0.f, 0.f);

        for (int p = 0; p < KP; ++p, ++it) {
            const int st = (int)(it & 1);
            if (pend[st]) {
                umma::mbar_wait(&bars[st], phase[st]);
                phase[st] ^= 1;
                pend[st] = false;
            }
            uint8_t* Ahi = smem + st * UM_STAGE;
            uint8_t* Alo = Ahi + UM_PANEL;
            uint8_t* Bhi = Alo + UM_PANEL;
            uint8_t* Blo = Bhi + UM_PANEL;
            // ---- stage operands
            if (MODE == UMMA_NN) {
                const int sp = p / (P.d_in / 32);
                const int kk = (p - sp * (P.d_in / 32)) * 32;
                const int64_t acol = (int64_t)sp * P.d_in + kk;
#pragma unroll
                for (int i = 0; i < 4; ++i) {           // A: 128 rows x 8 chunks, K-major
                    const int r = (tid >> 3) + 32 * i, c = tid & 7;
                    const int64_t row = row0 + r;
                    float4 v = (row < rlim) ? load4(P.A, P.lda, row, acol + 4 * c, acol + 32, vecA, nullptr)
                                            : make_float4(0.f, 0.f, 0.f, 0.f);
                    st_split(Ahi, Alo, umma::kmajor_off(r, 4 * c), v);
                }
                const float* W = P.B + (int64_t)rg.slot_w[t][sp] * P.bslot;
#pragma unroll
                for (int i = 0; i < 4; ++i) {           // B: rows k of W, MN = n, MN-major
                    const int kr = (tid >> 5) + 8 * i, j = tid & 31;
                    float4 v = load4(W, P.ldb, kk + kr, n0 + 4 * j, P.N, vecB, nullptr);
                    st_split(Bhi, Blo, umma::mnmajor_off(4 * j, kr), v);
                }
            } else if (MODE == UMMA_NT) {
                const int nn = p * 32;
#pragma unroll
                for (int i = 0; i < 4; ++i) {           // A: dZ rows, K = n, K-major
                    const int r = (tid >> 3) + 32 * i, c = tid & 7;
                    const int64_t row = row0 + r;
                    float4 v = (row < rlim) ? load4(P.A, P.lda, row, nn + 4 * c, P.N, vecA, P.relu ? P.H : nullptr)
                                            : make_float4(0.f, 0.f, 0.f, 0.f);
                    st_split(Ahi, Alo, umma::kmajor_off(r, 4 * c), v);
                }
                const float* W = P.B + (int64_t)rg.slot_w[t][s] * P.bslot;
#pragma unroll
                for (int i = 0; i < 4; ++i) {           // B: rows k of W (N' = k), K = n, K-major
                    const int r = (tid >> 3) + 32 * i, c = tid & 7;
                    const int k = c0 + r;
                    float4 v = (k < P.d_in) ? load4(W, P.ldb, k, nn + 4 * c, P.N, vecB, nullptr)
                                            : make_float4(0.f, 0.f, 0.f, 0.f);
                    st_split(Bhi, Blo, umma::kmajor_off(r, 4 * c), v);
                }
            } else {
                const int64_t rb = row0 + (int64_t)p * 32;
                const int64_t acol = (int64_t)s * P.d_in + c0;
#pragma unroll
                for (int i = 0; i < 4; ++i) {           // A': MN = k (Acat cols), K = rows, MN-major
                    const int kr = (tid >> 5) + 8 * i, j = tid & 31;
                    const int64_t row = rb + kr;
                    float4 v = (row < rlim) ? load4(P.A, P.lda, row, acol + 4 * j, (int64_t)s * P.d_in + P.d_in, vecA,
                                                    nullptr)
                                            : make_float4(0.f, 0.f, 0.f, 0.f);
                    st_split(Ahi, Alo, umma::mnmajor_off(4 * j, kr), v);
                }
#pragma unroll
                for (int i = 0; i < 4; ++i) {           // B': MN = n (dZ cols), K = rows, MN-major
                    const int kr = (tid >> 5) + 8 * i, j = tid & 31;
                    const int64_t row = rb + kr;
                    float4 v = (row < rlim) ? load4(P.B, P.ldb, row, n0 + 4 * j, P.N, vecB, P.relu ? P.H : nullptr)
                                            : make_float4(0.f, 0.f, 0.f, 0.f);
                    if (do_db) { cs.x += v.x; cs.y += v.y; cs.z += v.z; cs.w += v.w; }
                    st_split(Bhi, Blo, umma::mnmajor_off(4 * j, kr), v);
                }
            }
            umma::fence_proxy_async_smem();
            __syncthreads();
            if (tid == 0) {
                umma::tc_fence_after();
                const uint32_t a_hi = umma::smem_u32(Ahi), a_lo = umma::smem_u32(Alo);
                const uint32_t b_hi = umma::smem_u32(Bhi), b_lo = umma::smem_u32(Blo);
#pragma unroll
                for (int ks = 0; ks < 4; ++ks) {
                    const uint32_t oa = A_MN ? ks * 4096u : ks * 32u;
                    const uint32_t ob = B_MN ? ks * 4096u : ks * 32u;
                    const uint64_t dah = A_MN ? umma::desc_mnmajor(a_hi + oa) : umma::desc_kmajor(a_hi + oa);
                    const uint64_t dal = A_MN ? umma::desc_mnmajor(a_lo + oa) : umma::desc_kmajor(a_lo + oa);
                    const uint64_t dbh = B_MN ? umma::desc_mnmajor(b_hi + ob) : umma::desc_kmajor(b_hi + ob);
                    const uint64_t dbl = B_MN ? umma::desc_mnmajor(b_lo + ob) : umma::desc_kmajor(b_lo + ob);
                    umma::mma_tf32(tmem, dal, dbh, IDESC, (p > 0 || ks > 0) ? 1u : 0u);
                    umma::mma_tf32(tmem, dah, dbl, IDESC, 1u);
                    umma::mma_tf32(tmem, dah, dbh, IDESC, 1u);
                }
                umma::mma_commit(&bars[st]);
            }
            pend[st] = true;
        }
        // ---- drain the MMAs of this tile (older stage first)
        {
            const int last = (int)((it - 1) & 1), other = last ^ 1;
            if (pend[other]) { umma::mbar_wait(&bars[other], phase[other]); phase[other] ^= 1; pend[other] = false; }
            if (pend[last]) { umma::mbar_wait(&bars[last], phase[last]); phase[last] ^= 1; pend[last] = false; }
        }
        umma::tc_fence_after();
        // ---- epilogue: warp w reads TMEM lanes 32*(w&3).., columns half (w>>2)*64
        {
            const int q = warp & 3, half = warp >> 2;
            const int r = q * 32 + lane;
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) {
                const int col = half * 64 + cc * 32;
                float v[32];
                umma::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)col, v);
                if (MODE == UMMA_NN) {
                    const int64_t row = row0 + r;
                    if (row < rlim) {
                        float* out = P.C + row * P.ldc;
                        const bool vec = ((P.ldc & 3) == 0) && ((reinterpret_cast<uintptr_t>(P.C) & 15) == 0);
#pragma unroll
                        for (int e = 0; e < 32; e += 4) {
                            const int n = n0 + col + e;
                            float x[4];
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                x[u] = v[e + u] + ((P.bias && n + u < P.N) ? __ldg(P.bias + n + u) : 0.f);
                                if (P.relu) x[u] = fmaxf(x[u], 0.f);
                            }
                            if (vec && n + 3 < P.N) {
                                *reinterpret_cast<float4*>(out + n) = make_float4(x[0], x[1], x[2], x[3]);
                            } else {
                                for (int u = 0; u < 4; ++u)
                                    if (n + u < P.N) out[n + u] = x[u];
                            }
                        }
                    }
                } else if (MODE == UMMA_NT) {
                    const int64_t row = row0 + r;
                    if (row < rlim) {
                        float* out = P.C + row * P.ldc + (int64_t)s * P.d_in;
#pragma unroll
                        for (int e = 0; e < 32; ++e) {
                            const int k = c0 + col + e;
                            if (k < P.d_in) out[k] = v[e];
                        }
                    }
                } else {
                    const int k = c0 + r;
                    if (k < P.d_in) {
                        float* out = P.C + (int64_t)rg.slot_w[t][s] * P.bslot + (int64_t)k * P.ldc;
                        const bool vec = ((P.ldc & 3) == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
#pragma unroll
                        for (int e = 0; e < 32; e += 4) {
                            const int n = n0 + col + e;
                            if (vec && n + 3 < P.N) {
                                red_add_f4(out + n, make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]));
                            } else {
                                for (int u = 0; u < 4; ++u)
                                    if (n + u < P.N) atomicAdd(out + n + u, v[e + u]);
                            }
                        }
                    }
                }
            }
        }
        if (do_db) {   // column sums of dZ over the chunk (each thread owns 4 columns of 128)
            if (tid < 128) dbred[tid] = 0.f;
            __syncthreads();
            const int j = tid & 31;
            atomicAdd(&dbred[4 * j + 0], cs.x);
            atomicAdd(&dbred[4 * j + 1], cs.y);
            atomicAdd(&dbred[4 * j + 2], cs.z);
            atomicAdd(&dbred[4 * j + 3], cs.w);
            __syncthreads();
            if (tid < 128 && n0 + tid < P.N) atomicAdd(P.db + n0 + tid, dbred[tid]);
        }
        umma::tc_fence_before();
        __syncthreads();
    }
    umma::tc_fence_after();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc<128>(tmem);
}

template <int MODE>
inline gsb_status launch_umma(const char* name, const UProb& P, int64_t tiles_upper, cudaStream_t s) {
    static bool attr_set = false;
    if (!attr_set) {
        GSB_CUDA(cudaFuncSetAttribute(umma_gemm_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, UM_SMEM));
        attr_set = true;
    }
    int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles_upper, kNumSMs));
    GSB_LAUNCH(name, umma_gemm_kernel<MODE>, grid, UM_THREADS, UM_SMEM, s, P);
    return GSB_OK;
}

}  // namespace gsb
