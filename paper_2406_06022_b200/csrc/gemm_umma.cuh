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
#include "gsb_internal.cuh"
#include "umma.cuh"

namespace gsb {

// Row groups of a grouped GEMM: group t = the dst rows of ntype t (K-slots = its
// in-relations + self), or one plain group of M rows.
struct RowGroups {
    const HopMeta* meta;   // rows of group t = [meta->dst_off[t], meta->dst_off[t+1]) ; or
    int64_t M;             // meta == nullptr: one group [0, M)
    int32_t G;             // number of groups
    int32_t ks[kMaxT];     // K-slots of group t (in-relations + self)
    int32_t slot_w[kMaxT][kMaxS + 1];
};

__device__ __forceinline__ void group_rows(const RowGroups& rg, int t, int64_t& r0, int64_t& r1) {
    if (rg.meta) {
        r0 = rg.meta->dst_off[t];
        r1 = rg.meta->dst_off[t + 1];
    } else {
        r0 = 0;
        r1 = rg.M;
    }
}

constexpr int BK = 32;     // layer widths (d_in) are multiples of one 32-column tf32 panel

using umma::cp16;
using umma::cp4;
using umma::cp_commit;
using umma::cp_wait;

enum { UMMA_NN = 0, UMMA_NT = 1, UMMA_TN = 2 };

struct UProb {
    RowGroups rg;
    const float* A;        // NN: Acat/h ; NT: dH ; TN: Acat/h
    int64_t lda;
    const float* B;        // NN/NT: W ; TN: dH
    int64_t ldb;
    int64_t bslot;         // W slot stride (elements); 0 for a single matrix
    int relu;
    int d_in;              // K per slot (NN), output cols per slot (NT), output rows per slot (TN)
    int N;                 // output cols (NN, TN) / reduction length (NT)
    float* C;              // NN/NT output ; TN: dW
    int64_t ldc;
    const float* bias;     // NN
    float* db;             // TN (optional)
    int rows_per_chunk;    // TN
    int ksplit;            // NN/NT: K-panel splits per tile (>1: partials red.add into a zeroed C; no relu)
    int dbg;               // gemm_tma.cuh A/B knobs (GSB_GEMM_DBG): 1 no split, 2 no MMA, 4 no TMA
    int brow;              // gemm_tma.cuh: rows of B per weight slot (bslot / ldb)
    int bimg;              // gemm_tma.cuh: B comes pre-split (weight images, mapB = hi, mapB2 = lo)
    int cdirect;           // gemm_tma3.cuh: C is not TMA-addressable: per-thread stores / atomics
    int pf;                // gemm_tma3.cuh: L2 prefetch distance of the HBM-streamed operand panels
};

#ifndef GSB_UM_THREADS
#define GSB_UM_THREADS 256
#endif
constexpr int UM_THREADS = GSB_UM_THREADS;
constexpr int UM_NI = 1024 / UM_THREADS;      // 16-B chunks per thread per operand panel
constexpr int UM_RS = UM_THREADS / 8;         // K-major: row stride between a thread's chunks
constexpr int UM_KS = UM_THREADS / 32;        // MN-major: K-row stride between a thread's chunks
constexpr int UM_PANEL = 16384;            // bytes of one 128 x 32 fp32/tf32 panel
constexpr int UM_STAGE = 4 * UM_PANEL;     // A_hi(raw), A_lo, B_hi(raw), B_lo
constexpr int UM_STAGES = 3;
constexpr int UM_SMEM = UM_STAGES * UM_STAGE + 1024;

// Copy the 4 elements [c, c+4) of row `row` (cols >= ncols, rows out of range -> 0) to dst.
__device__ __forceinline__ void cp_chunk(uint32_t dst, const float* base, int64_t ld, int64_t row, bool row_ok,
                                         int64_t c, int64_t ncols, bool vec) {
    const float* src = base + (row_ok ? row * ld : 0);
    const int64_t valid = row_ok ? max((int64_t)0, min((int64_t)4, ncols - c)) : 0;
    if (vec) {
        cp16(dst, valid > 0 ? (const void*)(src + c) : (const void*)base, (int)(4 * valid));
    } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) cp4(dst + 4 * q, q < valid ? (const void*)(src + c + q) : (const void*)base,
                                        q < valid ? 4 : 0);
    }
}

__device__ __forceinline__ float4 lds128(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
    asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
// in-place split through 32-bit shared addresses (LDS/STS, not generic loads/stores)
__device__ __forceinline__ float4 split_chunk_s(uint32_t hi, uint32_t lo, uint32_t off) {
    const float4 v = lds128(hi + off);
    uint32_t h0, h1, h2, h3, l0, l1, l2, l3;
    umma::split_tf32(v.x, h0, l0);
    umma::split_tf32(v.y, h1, l1);
    umma::split_tf32(v.z, h2, l2);
    umma::split_tf32(v.w, h3, l3);
    sts128(hi + off, h0, h1, h2, h3);
    sts128(lo + off, l0, l1, l2, l3);
    return v;
}

// per-thread shared-memory offsets of its 4 A and 4 B chunks (constant for the kernel)
struct SmemOff {
    uint32_t a[UM_NI], b[UM_NI];
};
template <int MODE>
__device__ __forceinline__ SmemOff smem_offsets(int tid) {
    SmemOff o;
#pragma unroll
    for (int i = 0; i < UM_NI; ++i) {
        const uint32_t kmA = umma::kmajor_off((tid >> 3) + UM_RS * i, 4 * (tid & 7));
        const uint32_t mnA = umma::mnmajor_off(4 * (tid & 31), (tid >> 5) + UM_KS * i);
        o.a[i] = (MODE == UMMA_TN) ? mnA : kmA;
        o.b[i] = (MODE == UMMA_NT) ? kmA : mnA;
    }
    return o;
}


// One (tile, panel) position of this CTA's persistent schedule.
struct UCursor {
    int64_t tile;          // >= total: exhausted
    int p, KP;             // panels [p0, KP) of this (split) tile; p runs from p0
    int p0, split;
    int t, s, c0, n0;
    int64_t row0, rlim;
};

// K panels of one (NN / NT) tile of group t, and the split count used for that group: never
// more splits than panels, so every split owns a non-empty panel range [p0, p1).
template <int MODE>
__device__ __forceinline__ int panels_of_group(const UProb& P, int t) {
    return MODE == UMMA_NN ? P.rg.ks[t] * (P.d_in / 32) : (P.N + 31) / 32;
}
template <int MODE>
__device__ __forceinline__ int ksplit_of_group(const UProb& P, int t) {
    return max(1, min(P.ksplit, panels_of_group<MODE>(P, t)));
}

template <int MODE>
__device__ __forceinline__ int64_t tiles_of_group(const UProb& P, int t, int64_t r0, int64_t r1, int nct, int kct) {
    if (MODE == UMMA_NN) return ((r1 - r0 + 127) / 128) * nct * ksplit_of_group<MODE>(P, t);
    if (MODE == UMMA_NT) return ((r1 - r0 + 127) / 128) * kct * P.rg.ks[t] * ksplit_of_group<MODE>(P, t);
    return ((r1 - r0 + P.rows_per_chunk - 1) / P.rows_per_chunk) * P.rg.ks[t] * kct * nct;
}

template <int MODE>
__device__ __forceinline__ void decode_tile(const UProb& P, int64_t tile, int nct, int kct, UCursor& c) {
    const RowGroups& rg = P.rg;
    int t = 0;
    int64_t rem = tile, r0 = 0, r1 = 0;
    for (;; ++t) {
        group_rows(rg, t, r0, r1);
        const int64_t nt = tiles_of_group<MODE>(P, t, r0, r1, nct, kct);
        if (rem < nt) break;
        rem -= nt;
    }
    c.t = t;
    c.s = 0; c.c0 = 0; c.n0 = 0;
    c.split = 0;
    const int kse = (MODE != UMMA_TN) ? ksplit_of_group<MODE>(P, t) : 1;
    if (MODE != UMMA_TN) {
        c.split = (int)(rem % kse);
        rem /= kse;
    }
    if (MODE == UMMA_NN) {
        c.row0 = r0 + (rem / nct) * 128;
        c.rlim = r1;
        c.n0 = (int)(rem % nct) * 128;
        c.KP = rg.ks[t] * (P.d_in / 32);
    } else if (MODE == UMMA_NT) {
        const int per = kct * rg.ks[t];
        c.row0 = r0 + (rem / per) * 128;
        c.rlim = r1;
        const int q = (int)(rem % per);
        c.s = q / kct;
        c.c0 = (q % kct) * 128;
        c.KP = (P.N + 31) / 32;
    } else {
        const int per = rg.ks[t] * kct * nct;
        c.row0 = r0 + (rem / per) * P.rows_per_chunk;
        c.rlim = min(r1, c.row0 + (int64_t)P.rows_per_chunk);
        int q = (int)(rem % per);
        c.s = q / (kct * nct);
        q -= c.s * kct * nct;
        c.c0 = (q / nct) * 128;
        c.n0 = (q % nct) * 128;
        c.KP = (int)((c.rlim - c.row0 + 31) / 32);
    }
    c.p0 = 0;
    if (kse > 1) {   // split k owns panels [k*KP/kse, (k+1)*KP/kse): non-empty since kse <= KP
        const int kp = c.KP;
        c.p0 = (c.split * kp) / kse;
        c.KP = ((c.split + 1) * kp) / kse;
    }
    c.p = c.p0;
}

// issue this thread's cp.async copies of panel c.p into stage buffers (A: 4 chunks, B: 4 chunks)
template <int MODE>
__device__ __forceinline__ void issue_panel(const UProb& P, const UCursor& c, uint8_t* stage, int tid, bool vecA,
                                            bool vecB) {
    const uint32_t Ahi = umma::smem_u32(stage), Bhi = umma::smem_u32(stage + 2 * UM_PANEL);
    if (MODE == UMMA_NN) {
        const int per = P.d_in / 32;
        const int sp = c.p / per;
        const int kk = (c.p - sp * per) * 32;
        const int64_t acol = (int64_t)sp * P.d_in + kk;
#pragma unroll
        for (int i = 0; i < UM_NI; ++i) {
            const int r = (tid >> 3) + UM_RS * i, ch = tid & 7;
            const int64_t row = c.row0 + r;
            cp_chunk(Ahi + umma::kmajor_off(r, 4 * ch), P.A, P.lda, row, row < c.rlim, acol + 4 * ch, acol + 32, vecA);
        }
        const float* W = P.B + (int64_t)P.rg.slot_w[c.t][sp] * P.bslot;
#pragma unroll
        for (int i = 0; i < UM_NI; ++i) {
            const int kr = (tid >> 5) + UM_KS * i, j = tid & 31;
            cp_chunk(Bhi + umma::mnmajor_off(4 * j, kr), W, P.ldb, kk + kr, true, c.n0 + 4 * j, P.N, vecB);
        }
    } else if (MODE == UMMA_NT) {
        const int nn = c.p * 32;
#pragma unroll
        for (int i = 0; i < UM_NI; ++i) {
            const int r = (tid >> 3) + UM_RS * i, ch = tid & 7;
            const int64_t row = c.row0 + r;
            cp_chunk(Ahi + umma::kmajor_off(r, 4 * ch), P.A, P.lda, row, row < c.rlim, nn + 4 * ch, P.N, vecA);
        }
        const float* W = P.B + (int64_t)P.rg.slot_w[c.t][c.s] * P.bslot;
#pragma unroll
        for (int i = 0; i < UM_NI; ++i) {
            const int r = (tid >> 3) + UM_RS * i, ch = tid & 7;
            const int k = c.c0 + r;
            cp_chunk(Bhi + umma::kmajor_off(r, 4 * ch), W, P.ldb, k, k < P.d_in, nn + 4 * ch, P.N, vecB);
        }
    } else {
        const int64_t rb = c.row0 + (int64_t)c.p * 32;
        const int64_t acol = (int64_t)c.s * P.d_in + c.c0;
        const int64_t alim = (int64_t)c.s * P.d_in + P.d_in;
#pragma unroll
        for (int i = 0; i < UM_NI; ++i) {
            const int kr = (tid >> 5) + UM_KS * i, j = tid & 31;
            const int64_t row = rb + kr;
            cp_chunk(Ahi + umma::mnmajor_off(4 * j, kr), P.A, P.lda, row, row < c.rlim, acol + 4 * j, alim, vecA);
        }
#pragma unroll
        for (int i = 0; i < UM_NI; ++i) {
            const int kr = (tid >> 5) + UM_KS * i, j = tid & 31;
            const int64_t row = rb + kr;
            cp_chunk(Bhi + umma::mnmajor_off(4 * j, kr), P.B, P.ldb, row, row < c.rlim, c.n0 + 4 * j, P.N, vecB);
        }
    }
}

// Per-thread source pointers of the tile being loaded, resolved once per tile so that a panel's
// copies are a pointer add + cp.async each (the generic issue_panel recomputes row bases,
// slot weights and bounds for every chunk of every panel).  Used when all chunks are whole
// 16-B copies (aligned operands, N / d_in multiples of 4 or 32 as below).
struct FastSrc {
    const float* a[UM_NI];
    const float* b[UM_NI];
    int64_t arow[UM_NI];     // TN: first row of this thread's A/B chunk rows (row0 + kr)
    int64_t boff[UM_NI];     // NN: element offset of this thread's B chunks inside a W slot panel
    bool bok;            // NN: this thread's B columns exist
};

template <int MODE>
__device__ __forceinline__ void fast_setup(const UProb& P, const UCursor& c, int tid, FastSrc& f) {
    if (MODE == UMMA_NN) {
        const int ch = tid & 7, j = tid & 31;
#pragma unroll
        for (int i = 0; i < UM_NI; ++i) {
            const int64_t row = c.row0 + (tid >> 3) + UM_RS * i;
            f.a[i] = row < c.rlim ? P.A + row * P.lda + 4 * ch : nullptr;
            const int kr = (tid >> 5) + UM_KS * i;
            f.boff[i] = (int64_t)kr * P.ldb + c.n0 + 4 * j;
        }
        f.bok = c.n0 + 4 * j < P.N;
    } else if (MODE == UMMA_NT) {
        const int ch = tid & 7;
        const float* W = P.B + (int64_t)P.rg.slot_w[c.t][c.s] * P.bslot;
#pragma unroll
        for (int i = 0; i < UM_NI; ++i) {
            const int r = (tid >> 3) + UM_RS * i;
            const int64_t row = c.row0 + r;
            f.a[i] = row < c.rlim ? P.A + row * P.lda + 4 * ch : nullptr;
            const int k = c.c0 + r;
            f.b[i] = k < P.d_in ? W + (int64_t)k * P.ldb + 4 * ch : nullptr;
        }
    } else {
        const int j = tid & 31;
        const int64_t acol = (int64_t)c.s * P.d_in + c.c0 + 4 * j;
        const bool aok = c.c0 + 4 * j < P.d_in, bok = c.n0 + 4 * j < P.N;
#pragma unroll
        for (int i = 0; i < UM_NI; ++i) {
            const int64_t row = c.row0 + (tid >> 5) + UM_KS * i;
            f.arow[i] = row;
            f.a[i] = aok ? P.A + row * P.lda + acol : nullptr;
            f.b[i] = bok ? P.B + row * P.ldb + c.n0 + 4 * j : nullptr;
        }
    }
}

template <int MODE>
__device__ __forceinline__ void issue_panel_fast(const UProb& P, const UCursor& c, const FastSrc& f,
                                                 const SmemOff& so, uint32_t Ahi) {
    const uint32_t Bhi = Ahi + 2 * UM_PANEL;
    if (MODE == UMMA_NN) {
        const int per = P.d_in / 32;
        const int sp = c.p / per;
        const int kk = (c.p - sp * per) * 32;
        const float* W = P.B + (int64_t)P.rg.slot_w[c.t][sp] * P.bslot + (int64_t)kk * P.ldb;
#pragma unroll
        for (int i = 0; i < UM_NI; ++i) {
            cp16(Ahi + so.a[i], f.a[i] ? f.a[i] + c.p * 32 : P.A, f.a[i] ? 16 : 0);
            cp16(Bhi + so.b[i], f.bok ? W + f.boff[i] : P.B, f.bok ? 16 : 0);
        }
    } else if (MODE == UMMA_NT) {
#pragma unroll
        for (int i = 0; i < UM_NI; ++i) {
            cp16(Ahi + so.a[i], f.a[i] ? f.a[i] + c.p * 32 : P.A, f.a[i] ? 16 : 0);
            cp16(Bhi + so.b[i], f.b[i] ? f.b[i] + c.p * 32 : P.B, f.b[i] ? 16 : 0);
        }
    } else {
        const int64_t dr = (int64_t)c.p * 32;
#pragma unroll
        for (int i = 0; i < UM_NI; ++i) {
            const bool rok = f.arow[i] + dr < c.rlim;
            const bool oa = rok && f.a[i], ob = rok && f.b[i];
            cp16(Ahi + so.a[i], oa ? f.a[i] + dr * P.lda : P.A, oa ? 16 : 0);
            cp16(Bhi + so.b[i], ob ? f.b[i] + dr * P.ldb : P.B, ob ? 16 : 0);
        }
    }
}

// split this thread's own chunks of a landed stage (shared addresses, precomputed offsets)
template <int MODE>
__device__ __forceinline__ float4 split_panel_s(uint32_t stage, const SmemOff& so) {
    float4 cs = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int i = 0; i < UM_NI; ++i) split_chunk_s(stage, stage + UM_PANEL, so.a[i]);
#pragma unroll
    for (int i = 0; i < UM_NI; ++i) {
        const float4 v = split_chunk_s(stage + 2 * UM_PANEL, stage + 3 * UM_PANEL, so.b[i]);
        cs.x += v.x; cs.y += v.y; cs.z += v.z; cs.w += v.w;
    }
    return cs;
}

template <int MODE>
__global__ void __launch_bounds__(UM_THREADS, 1) umma_gemm_kernel(UProb P) {
    GSB_PDL_ENTRY();
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
    const bool fast = vecA && vecB && ((P.bslot & 3) == 0) &&
                      (MODE == UMMA_NN ? (P.N & 3) == 0 : MODE == UMMA_NT ? (P.N & 31) == 0
                                                                          : ((P.N & 3) == 0 && (P.d_in & 3) == 0));
    FastSrc fs;

    const int nct = (P.N + 127) / 128;
    const int kct = (P.d_in + 127) / 128;
    int64_t total = 0;
    for (int t = 0; t < rg.G; ++t) {
        int64_t r0, r1;
        group_rows(rg, t, r0, r1);
        total += tiles_of_group<MODE>(P, t, r0, r1, nct, kct);
    }

    // two cursors over the same (tile, panel) sequence: loads run UM_STAGES-1 panels ahead
    UCursor ld, cp;
    ld.tile = blockIdx.x;
    if (ld.tile < total) {
        decode_tile<MODE>(P, ld.tile, nct, kct, ld);
        if (fast) fast_setup<MODE>(P, ld, tid, fs);
    }
    cp = ld;
    auto advance = [&](UCursor& c, bool is_ld) {
        if (c.tile >= total) return;
        if (++c.p >= c.KP) {
            c.tile += gridDim.x;
            if (c.tile < total) {
                decode_tile<MODE>(P, c.tile, nct, kct, c);
                if (is_ld && fast) fast_setup<MODE>(P, c, tid, fs);
            }
        }
    };
    const SmemOff so = smem_offsets<MODE>(tid);
    auto issue = [&](uint8_t* stage) {
        if (fast) issue_panel_fast<MODE>(P, ld, fs, so, umma::smem_u32(stage));
        else issue_panel<MODE>(P, ld, stage, tid, vecA, vecB);
    };
    uint32_t phase = 0, pend = 0;          // per-stage bits
    int st_ld = 0, st_cp = 0;              // stage of the next load / of the panel being computed
    auto wait_stage = [&](int st) {
        if (pend & (1u << st)) {
            umma::mbar_wait(&bars[st], (phase >> st) & 1u);
            phase ^= 1u << st;
            pend &= ~(1u << st);
        }
    };
    auto next_st = [](int s) { return s + 1 == UM_STAGES ? 0 : s + 1; };
    // prologue
    for (int k = 0; k < UM_STAGES - 1; ++k) {
        if (ld.tile < total) {
            issue(smem + st_ld * UM_STAGE);
            advance(ld, true);
        }
        cp_commit();
        st_ld = next_st(st_ld);
    }
    float4 cs = make_float4(0.f, 0.f, 0.f, 0.f);
    while (cp.tile < total) {
        // data of panel it_cp landed (the one newer group may still be in flight)
        cp_wait<UM_STAGES - 2>();
        const int st = st_cp;
        uint8_t* stage = smem + st * UM_STAGE;
        const bool do_db = (MODE == UMMA_TN) && P.db && (cp.s == rg.ks[cp.t] - 1) && cp.c0 == 0;
        {   // split overlaps the tensor pipe still working on the previous panel
            float4 v = split_panel_s<MODE>(umma::smem_u32(stage), so);
            if (do_db) { cs.x += v.x; cs.y += v.y; cs.z += v.z; cs.w += v.w; }
        }
        umma::fence_proxy_async_smem();
        __syncthreads();
        if (tid == 0) {
            umma::tc_fence_after();
            const uint32_t a_hi = umma::smem_u32(stage), a_lo = a_hi + UM_PANEL;
            const uint32_t b_hi = a_hi + 2 * UM_PANEL, b_lo = a_hi + 3 * UM_PANEL;
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                const uint32_t oa = A_MN ? ks * 4096u : ks * 32u;
                const uint32_t ob = B_MN ? ks * 4096u : ks * 32u;
                const uint64_t dah = A_MN ? umma::desc_mnmajor(a_hi + oa) : umma::desc_kmajor(a_hi + oa);
                const uint64_t dal = A_MN ? umma::desc_mnmajor(a_lo + oa) : umma::desc_kmajor(a_lo + oa);
                const uint64_t dbh = B_MN ? umma::desc_mnmajor(b_hi + ob) : umma::desc_kmajor(b_hi + ob);
                const uint64_t dbl = B_MN ? umma::desc_mnmajor(b_lo + ob) : umma::desc_kmajor(b_lo + ob);
                umma::mma_tf32(tmem, dal, dbh, IDESC, (cp.p > cp.p0 || ks > 0) ? 1u : 0u);
                umma::mma_tf32(tmem, dah, dbl, IDESC, 1u);
                umma::mma_tf32(tmem, dah, dbh, IDESC, 1u);
            }
            umma::mma_commit(&bars[st]);
        }
        pend |= 1u << st;
        // refill: the stage of panel it_cp-1 receives panel it_cp+2 once its MMAs are done
        {
            const int fst = st_ld;
            wait_stage(fst);
            if (ld.tile < total) {
                issue(smem + fst * UM_STAGE);
                advance(ld, true);
            }
            cp_commit();
            st_ld = next_st(st_ld);
        }
        st_cp = next_st(st_cp);
        if (cp.p + 1 < cp.KP) {
            advance(cp, false);
            continue;
        }
        // ---- last panel of the tile: drain its MMAs, then the epilogue
        {
            int w = st_cp;                                   // oldest pending stage first
            for (int k = 0; k < UM_STAGES; ++k, w = next_st(w)) wait_stage(w);
        }
        umma::tc_fence_after();
        {
            constexpr int CW = 128 / (UM_THREADS / 128);   // columns drained per warp
            const int q = warp & 3, half = warp >> 2;
            const int r = q * 32 + lane;
#pragma unroll
            for (int cc = 0; cc < CW / 32; ++cc) {
                const int col = half * CW + cc * 32;
                float v[32];
                umma::tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)col, v);
                if (MODE == UMMA_NN && P.ksplit > 1) {
                    const int64_t row = cp.row0 + r;
                    if (row < cp.rlim) {
                        float* out = P.C + row * P.ldc;
                        const bool vec = ((P.ldc & 3) == 0) && ((reinterpret_cast<uintptr_t>(P.C) & 15) == 0);
#pragma unroll
                        for (int e = 0; e < 32; e += 4) {
                            const int n = cp.n0 + col + e;
                            float x[4];
#pragma unroll
                            for (int u = 0; u < 4; ++u)
                                x[u] = v[e + u] + ((cp.split == 0 && P.bias && n + u < P.N) ? __ldg(P.bias + n + u) : 0.f);
                            if (vec && n + 3 < P.N) {
                                red_add_f4(out + n, make_float4(x[0], x[1], x[2], x[3]));
                            } else {
                                for (int u = 0; u < 4; ++u)
                                    if (n + u < P.N) atomicAdd(out + n + u, x[u]);
                            }
                        }
                    }
                } else if (MODE == UMMA_NN) {
                    const int64_t row = cp.row0 + r;
                    if (row < cp.rlim) {
                        float* out = P.C + row * P.ldc;
                        const bool vec = ((P.ldc & 3) == 0) && ((reinterpret_cast<uintptr_t>(P.C) & 15) == 0);
#pragma unroll
                        for (int e = 0; e < 32; e += 4) {
                            const int n = cp.n0 + col + e;
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
                    const int64_t row = cp.row0 + r;
                    if (row < cp.rlim) {
                        float* out = P.C + row * P.ldc + (int64_t)cp.s * P.d_in;
                        const bool vec = ((P.ldc & 3) == 0) && ((P.d_in & 3) == 0) &&
                                         ((reinterpret_cast<uintptr_t>(P.C) & 15) == 0);
#pragma unroll
                        for (int e = 0; e < 32; e += 4) {
                            const int k = cp.c0 + col + e;
                            if (P.ksplit > 1) {
                                if (vec && k + 3 < P.d_in) {
                                    red_add_f4(out + k, make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]));
                                } else {
                                    for (int u = 0; u < 4; ++u)
                                        if (k + u < P.d_in) atomicAdd(out + k + u, v[e + u]);
                                }
                            } else if (vec && k + 3 < P.d_in) {
                                *reinterpret_cast<float4*>(out + k) = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
                            } else {
                                for (int u = 0; u < 4; ++u)
                                    if (k + u < P.d_in) out[k + u] = v[e + u];
                            }
                        }
                    }
                } else {
                    const int k = cp.c0 + r;
                    if (k < P.d_in) {
                        float* out = P.C + (int64_t)rg.slot_w[cp.t][cp.s] * P.bslot + (int64_t)k * P.ldc;
                        const bool vec = ((P.ldc & 3) == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
#pragma unroll
                        for (int e = 0; e < 32; e += 4) {
                            const int n = cp.n0 + col + e;
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
        if (do_db) {   // column sums of dZ over the chunk (thread owns columns 4*(tid&31)..+3)
            if (tid < 128) dbred[tid] = 0.f;
            __syncthreads();
            const int j = tid & 31;
            atomicAdd(&dbred[4 * j + 0], cs.x);
            atomicAdd(&dbred[4 * j + 1], cs.y);
            atomicAdd(&dbred[4 * j + 2], cs.z);
            atomicAdd(&dbred[4 * j + 3], cs.w);
            __syncthreads();
            if (tid < 128 && cp.n0 + tid < P.N) atomicAdd(P.db + cp.n0 + tid, dbred[tid]);
        }
        cs = make_float4(0.f, 0.f, 0.f, 0.f);
        umma::tc_fence_before();
        __syncthreads();
        advance(cp, false);
    }
    cp_wait<0>();
    umma::tc_fence_after();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc<128>(tmem);
}

// Split-K choice for NN/NT: when a problem has too few output tiles to fill the SMs, split
// each tile's K panels (>= 3 panels per split) across CTAs.  Split outputs are accumulated
// with red.add, so C must be zeroed first and relu is not allowed (callers check).
inline int choose_ksplit(int64_t tiles_upper, int kp, bool allowed) {
    if (!allowed || tiles_upper * 2 > kNumSMs) return 1;
    int k = (int)std::min<int64_t>(kNumSMs / std::max<int64_t>(tiles_upper, 1), (kp + 2) / 3);
    return std::max(1, k);
}

template <int MODE>
inline gsb_status launch_umma(const char* name, UProb P, int64_t tiles_upper, cudaStream_t s) {
    static bool attr_set = false;
    if (!attr_set) {
        GSB_CUDA(cudaFuncSetAttribute(umma_gemm_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, UM_SMEM));
        attr_set = true;
    }
    if (P.ksplit < 1) P.ksplit = 1;
    int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles_upper * P.ksplit, kNumSMs));
    GSB_LAUNCH(name, umma_gemm_kernel<MODE>, grid, UM_THREADS, UM_SMEM, s, P);
    return GSB_OK;
}

}  // namespace gsb
