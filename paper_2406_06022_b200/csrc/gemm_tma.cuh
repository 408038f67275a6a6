// gemm_tma.cuh -- the grouped RGCN GEMMs (modes NN / NT / TN of gemm_umma.cuh, same tile
// schedule and epilogues) as a warp-specialized tcgen05 pipeline fed by TMA.
//
//   warp 0      TMA producer: one thread issues cp.async.bulk.tensor loads of the raw fp32
//               operand panels (A 128 x 32, B 32 x 128 or 128 x 32) into a 3-deep raw ring,
//               completion by mbarrier transaction count.  Never waits on the math.
//   warps 2-5   splitters: raw fp32 -> tf32 hi + lo (3xTF32) into a 2-deep MMA ring, in the
//               UMMA layouts (K-major SWIZZLE_128B is TMA's own layout: split in place of
//               position; MN-major operands are re-laid into SWIZZLE_128B_BASE32B).  TN: rows
//               past the group end are zeroed here, and the bias gradient (column sums of dZ)
//               is accumulated from the values being split.
//   warp 1      TMEM owner + MMA issuer: 4 k-steps x 3 tcgen05.mma.kind::tf32 per panel into
//               one of two 128-column TMEM accumulators; tcgen05.commit frees the MMA stage
//               and, after a tile's last panel, hands the accumulator to the epilogue.
//   warps 6-9   epilogue: tcgen05.ld of the accumulator (warp w reads TMEM lanes
//               32*(w%4)..+31), bias / ReLU / store, split-K and weight-gradient red.add.
//
// Versus gemm_umma.cuh (all 256 threads load with cp.async, split, and wait for the MMAs of
// the stage they refill), loads run up to 3 panels ahead of the splitters and the MMA ring
// is double-buffered, so HBM/L2 latency, the split and the tensor pipe overlap.
#pragma once
#include <cuda.h>

#include "gemm_umma.cuh"

namespace gsb {

namespace tma {

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(umma::smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(umma::smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void load_2d(uint32_t dst, const CUtensorMap* map, int32_t c0, int32_t c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(umma::smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
// wait for a phase with a nanosleep back-off between polls (threads that wait long, e.g. the
// epilogue during a whole mainloop, then do not steal issue slots from the working warps)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
    const uint32_t a = umma::smem_u32(bar);
    uint32_t done = 0, ns = 32;
    for (;;) {
        asm volatile(
            "{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.u32 %0, 1, 0, "
            "P1;\n\t}"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
        if (done) return;
        __nanosleep(ns);
        if (ns < 256) ns <<= 1;
    }
}
// poll with test_wait (never suspends) or try_wait (may suspend the thread until the phase
// completes or a system time limit passes)
__device__ __forceinline__ void mbar_wait_k(uint64_t* bar, uint32_t parity, bool test) {
    if (!test) {
        umma::mbar_wait(bar, parity);
        return;
    }
    const uint32_t a = umma::smem_u32(bar);
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "TW_%=:\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra TW_%=;\n\t}" ::"r"(a),
        "r"(parity)
        : "memory");
}
// one lane polls, the warp follows (fewer spinning threads)
__device__ __forceinline__ void mbar_wait_warp(uint64_t* bar, uint32_t parity) {
    if ((threadIdx.x & 31) == 0) umma::mbar_wait(bar, parity);
    __syncwarp();
}
__device__ __forceinline__ void named_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

}  // namespace tma

// dbg & 1024: CTA 0 records globaltimer stamps per role per panel (tools; gsb_gemm_trace)
constexpr int TG_TRACE = 64;
__device__ unsigned long long g_gemm_trace[4][TG_TRACE];
__device__ __forceinline__ void trace_mark(const UProb& P, int role, int i) {
    if ((P.dbg & 1024) && blockIdx.x == 0 && i < TG_TRACE) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        g_gemm_trace[role][i] = t;
    }
}

#ifndef GSB_TG_SPLIT_WARPS
#define GSB_TG_SPLIT_WARPS 8
#endif
// splitter warps: the split is latency / smem bound (more warps split faster) but every thread
// of this one-CTA-per-SM kernel holds its registers for the whole launch, and the sample phase
// of the next batch runs concurrently on the same SMs (profiles/round2_gemm_split_warps.md)
constexpr int TG_SPLIT_WARPS = GSB_TG_SPLIT_WARPS;
constexpr int TG_SPLIT = 32 * TG_SPLIT_WARPS;     // splitter threads
constexpr int TG_EPI_WARP0 = 2 + TG_SPLIT_WARPS;  // first epilogue warp
constexpr int TG_THREADS = 32 * (TG_EPI_WARP0 + 4);
constexpr int TG_PER = 1024 / TG_SPLIT;           // float4 of one operand panel per splitter thread
constexpr int TG_RAW = 3, TG_MMA = 2;           // ring depths
constexpr int TG_RAW_STAGE = 2 * UM_PANEL;      // A raw + B raw (32 KB)
constexpr int TG_MMA_STAGE = 4 * UM_PANEL;      // A hi, A lo, B hi, B lo (64 KB)
constexpr int TG_SMEM = TG_RAW * TG_RAW_STAGE + TG_MMA * TG_MMA_STAGE + 1024;

// split this thread's TG_PER float4 of one 16 KB operand panel at precomputed byte offsets:
// src[i] in the raw panel, dst[i] in the hi / lo panels.  K-major operands: the raw panel
// already has the UMMA K-major layout (TMA SWIZZLE_128B), so dst = src; MN-major operands: the
// raw panel is plain row-major [32 k][128 mn] fp32, re-laid into SWIZZLE_128B_BASE32B.  ZERO:
// rows k (kr[i]) with k >= klim are zeroed (TN: rows past the group); the column sums of the
// values split are returned (TN bias gradient).
template <bool ZERO>
__device__ __forceinline__ float4 split_panel_tma(uint32_t raw, uint32_t hi, uint32_t lo, const uint32_t (&src)[TG_PER],
                                                  const uint32_t (&dst)[TG_PER], const int (&kr)[TG_PER], int klim) {
    float4 cs = make_float4(0.f, 0.f, 0.f, 0.f);
    float4 v[TG_PER];
#pragma unroll
    for (int i = 0; i < TG_PER; ++i) v[i] = lds128(raw + src[i]);
#pragma unroll
    for (int i = 0; i < TG_PER; ++i) {
        if (ZERO) {
            if (kr[i] >= klim) v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            cs.x += v[i].x; cs.y += v[i].y; cs.z += v[i].z; cs.w += v[i].w;
        }
        uint32_t h0, h1, h2, h3, l0, l1, l2, l3;
        umma::split_tf32(v[i].x, h0, l0);
        umma::split_tf32(v[i].y, h1, l1);
        umma::split_tf32(v[i].z, h2, l2);
        umma::split_tf32(v[i].w, h3, l3);
        sts128(hi + dst[i], h0, h1, h2, h3);
        sts128(lo + dst[i], l0, l1, l2, l3);
    }
    return cs;
}

// Coordinates (innermost first) of panel c.p of the current tile, for the A and B maps.
template <int MODE>
__device__ __forceinline__ void panel_coords(const UProb& P, const UCursor& c, int32_t& a0, int32_t& a1, int32_t& b0,
                                             int32_t& b1) {
    if (MODE == UMMA_NN) {          // A = Acat [rows][lda] K-major ; B = W [(slots) d_in][N] plain
        const int per = P.d_in / 32;
        const int sp = c.p / per;
        const int kk = (c.p - sp * per) * 32;
        a0 = sp * P.d_in + kk;
        a1 = (int32_t)c.row0;
        if (P.bimg) {               // weight image W^T [(slots) N][K]: K-major, brow = N
            b0 = kk;
            b1 = P.rg.slot_w[c.t][sp] * P.brow + c.n0;
        } else {
            b0 = c.n0;
            b1 = P.rg.slot_w[c.t][sp] * P.brow + kk;
        }
    } else if (MODE == UMMA_NT) {   // A = dZ [rows][N] K-major ; B = W [(slots) d_in][N] K-major
        a0 = c.p * 32;
        a1 = (int32_t)c.row0;
        b0 = c.p * 32;
        b1 = P.rg.slot_w[c.t][c.s] * P.brow + c.c0;
    } else {                        // TN: A = Acat [rows][lda] plain ; B = dZ [rows][N] plain
        const int64_t rb = c.row0 + (int64_t)c.p * 32;
        a0 = c.s * P.d_in + c.c0;
        a1 = (int32_t)rb;
        b0 = c.n0;
        b1 = (int32_t)rb;
    }
}

template <int MODE>
__device__ __forceinline__ int64_t total_tiles(const UProb& P, int nct, int kct) {
    int64_t total = 0;
    for (int t = 0; t < P.rg.G; ++t) {
        int64_t r0, r1;
        group_rows(P.rg, t, r0, r1);
        total += tiles_of_group<MODE>(P, t, r0, r1, nct, kct);
    }
    return total;
}

template <int MODE>
__global__ void __launch_bounds__(TG_THREADS, 1) tma_gemm_kernel(const __grid_constant__ CUtensorMap mapA,
                                                                  const __grid_constant__ CUtensorMap mapB,
                                                                  const __grid_constant__ CUtensorMap mapB2, UProb P) {
    GSB_PDL_ENTRY();
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* raw_ring = smem;
    uint8_t* mma_ring = smem + TG_RAW * TG_RAW_STAGE;
    __shared__ __align__(8) uint64_t raw_full[TG_RAW], raw_empty[TG_RAW], mma_full[TG_MMA], mma_empty[TG_MMA];
    __shared__ __align__(8) uint64_t acc_full[2], acc_empty[2];
    __shared__ uint32_t tmem_sh;
    __shared__ float dbred[128];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    if (tid == 0) {
        for (int s = 0; s < TG_RAW; ++s) {
            umma::mbar_init(&raw_full[s], 1);
            umma::mbar_init(&raw_empty[s], TG_SPLIT_WARPS);
        }
        for (int s = 0; s < TG_MMA; ++s) {
            umma::mbar_init(&mma_full[s], TG_SPLIT_WARPS + (P.bimg ? 1 : 0));
            umma::mbar_init(&mma_empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            umma::mbar_init(&acc_full[s], 1);
            umma::mbar_init(&acc_empty[s], 4);
        }
        umma::fence_barrier_init();
        tma::prefetch_map(&mapA);
        tma::prefetch_map(&mapB);
        if (P.bimg) tma::prefetch_map(&mapB2);
    }
    if (tid < 128) dbred[tid] = 0.f;
    if (warp == 1) umma::tmem_alloc<256>(&tmem_sh);
    umma::tc_fence_before();
    __syncthreads();
    umma::tc_fence_after();
    const uint32_t tmem = tmem_sh;

    const int nct = (P.N + 127) / 128;
    const int kct = (P.d_in + 127) / 128;
    const int64_t total = (P.dbg & 64) ? 0 : total_tiles<MODE>(P, nct, kct);
    constexpr bool A_MN = (MODE == UMMA_TN);
    const bool B_MN = (MODE == UMMA_TN) || (MODE == UMMA_NN && !P.bimg);

    UCursor c;
    c.tile = blockIdx.x;
    if (c.tile < total) decode_tile<MODE>(P, c.tile, nct, kct, c);
    auto advance = [&](UCursor& u) {
        if (u.tile >= total) return;
        if (++u.p >= u.KP) {
            u.tile += gridDim.x;
            if (u.tile < total) decode_tile<MODE>(P, u.tile, nct, kct, u);
        }
    };

    if (tid == 0) trace_mark(P, 0, TG_TRACE - 1);
    if (warp == 0) {
        // ------------------------------------------------------------- TMA producer
        if (lane == 0) {
            int rs = 0, pi = 0;
            uint32_t rph = 0;
            while (c.tile < total) {
                tma::mbar_wait_k(&raw_empty[rs], rph ^ 1u, P.dbg & 512);
                int32_t a0, a1, b0, b1;
                panel_coords<MODE>(P, c, a0, a1, b0, b1);
                const uint32_t dst = umma::smem_u32(raw_ring + rs * TG_RAW_STAGE);
                if (P.dbg & 4) {
                    tma::mbar_arrive(&raw_full[rs]);
                } else if (P.bimg) {            // A only: B goes straight into the MMA ring (lane 1)
                    tma::mbar_expect_tx(&raw_full[rs], UM_PANEL);
                    tma::load_2d(dst, &mapA, a0, a1, &raw_full[rs]);
                } else {
                    tma::mbar_expect_tx(&raw_full[rs], TG_RAW_STAGE);
                    tma::load_2d(dst, &mapA, a0, a1, &raw_full[rs]);
                    tma::load_2d(dst + UM_PANEL, &mapB, b0, b1, &raw_full[rs]);
                }
                trace_mark(P, 0, pi++);
                if (++rs == TG_RAW) { rs = 0; rph ^= 1u; }
                advance(c);
            }
        } else if (lane == 1 && P.bimg) {
            // pre-split weights: the hi / lo panels are TMA'd into the MMA stage once the MMAs of
            // the panel two back have drained it; the splitters only split A
            int ms = 0;
            uint32_t mph = 0;
            while (c.tile < total) {
                tma::mbar_wait_k(&mma_empty[ms], mph ^ 1u, false);
                int32_t a0, a1, b0, b1;
                panel_coords<MODE>(P, c, a0, a1, b0, b1);
                const uint32_t mm = umma::smem_u32(mma_ring + ms * TG_MMA_STAGE);
                tma::mbar_expect_tx(&mma_full[ms], 2 * UM_PANEL);
                tma::load_2d(mm + 2 * UM_PANEL, &mapB, b0, b1, &mma_full[ms]);
                tma::load_2d(mm + 3 * UM_PANEL, &mapB2, b0, b1, &mma_full[ms]);
                if (++ms == TG_MMA) { ms = 0; mph ^= 1u; }
                advance(c);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------- MMA issuer
        if (lane == 0) {
            const uint32_t IDESC = umma::idesc_tf32(128, A_MN, B_MN);
            int ms = 0, as = 0, pi = 0;
            uint32_t mph = 0, aph = 0;
            while (c.tile < total) {
                if (c.p == c.p0) {          // first panel of a tile: the accumulator must be drained
                    tma::mbar_wait_k(&acc_empty[as], aph ^ 1u, P.dbg & 512);
                    umma::tc_fence_after();
                }
                tma::mbar_wait_k(&mma_full[ms], mph, P.dbg & 512);
                umma::tc_fence_after();
                const uint32_t a_hi = umma::smem_u32(mma_ring + ms * TG_MMA_STAGE), a_lo = a_hi + UM_PANEL;
                const uint32_t b_hi = a_hi + 2 * UM_PANEL, b_lo = a_hi + 3 * UM_PANEL;
                const uint32_t d = tmem + (uint32_t)(as * 128);
#pragma unroll
                for (int ks = 0; ks < ((P.dbg & 2) ? 0 : 4); ++ks) {
                    const uint32_t oa = A_MN ? ks * 4096u : ks * 32u;
                    const uint32_t ob = B_MN ? ks * 4096u : ks * 32u;
                    const uint64_t dah = A_MN ? umma::desc_mnmajor(a_hi + oa) : umma::desc_kmajor(a_hi + oa);
                    const uint64_t dal = A_MN ? umma::desc_mnmajor(a_lo + oa) : umma::desc_kmajor(a_lo + oa);
                    const uint64_t dbh = B_MN ? umma::desc_mnmajor(b_hi + ob) : umma::desc_kmajor(b_hi + ob);
                    const uint64_t dbl = B_MN ? umma::desc_mnmajor(b_lo + ob) : umma::desc_kmajor(b_lo + ob);
                    umma::mma_tf32(d, dal, dbh, IDESC, (c.p > c.p0 || ks > 0) ? 1u : 0u);
                    umma::mma_tf32(d, dah, dbl, IDESC, 1u);
                    umma::mma_tf32(d, dah, dbh, IDESC, 1u);
                }
                trace_mark(P, 1, pi++);
                if (P.dbg & 32) tma::mbar_arrive(&mma_empty[ms]);
                else umma::mma_commit(&mma_empty[ms]);
                if (++ms == TG_MMA) { ms = 0; mph ^= 1u; }
                if (c.p + 1 == c.KP) {
                    if (P.dbg & 32) tma::mbar_arrive(&acc_full[as]);
                    else umma::mma_commit(&acc_full[as]);
                    if (++as == 2) { as = 0; aph ^= 1u; }
                }
                advance(c);
            }
        }
    } else if (warp < TG_EPI_WARP0) {
        // ------------------------------------------------------------- splitters
        const int t = tid - 64;
        uint32_t offK[TG_PER], offM[TG_PER];
        int kr[TG_PER];
#pragma unroll
        for (int i = 0; i < TG_PER; ++i) {
            const int j = t + TG_SPLIT * i;        // float4 index in the panel
            offK[i] = 16u * j;
            kr[i] = j >> 5;                        // plain [32][128] panel: row k, columns 4*(j&31)..+3
            offM[i] = umma::mnmajor_off(4 * (j & 31), kr[i]);
        }
        int rs = 0, ms = 0, pi = 0;
        uint32_t rph = 0, mph = 0;
        float4 cs = make_float4(0.f, 0.f, 0.f, 0.f);
        while (c.tile < total) {
            tma::mbar_wait_k(&raw_full[rs], rph, P.dbg & 512);
            tma::mbar_wait_k(&mma_empty[ms], mph ^ 1u, P.dbg & 512);
            const uint32_t raw = umma::smem_u32(raw_ring + rs * TG_RAW_STAGE);
            const uint32_t mm = umma::smem_u32(mma_ring + ms * TG_MMA_STAGE);
            if (P.dbg & 1) {
            } else if (MODE == UMMA_TN) {
                const int klim = (int)min((int64_t)32, c.rlim - (c.row0 + (int64_t)c.p * 32));
                split_panel_tma<true>(raw, mm, mm + UM_PANEL, offK, offM, kr, klim);
                const float4 v = split_panel_tma<true>(raw + UM_PANEL, mm + 2 * UM_PANEL, mm + 3 * UM_PANEL, offK,
                                                       offM, kr, klim);
                cs.x += v.x; cs.y += v.y; cs.z += v.z; cs.w += v.w;
            } else {
                split_panel_tma<false>(raw, mm, mm + UM_PANEL, offK, offK, kr, 32);
                if (P.bimg) {
                } else if (MODE == UMMA_NN)
                    split_panel_tma<false>(raw + UM_PANEL, mm + 2 * UM_PANEL, mm + 3 * UM_PANEL, offK, offM, kr, 32);
                else
                    split_panel_tma<false>(raw + UM_PANEL, mm + 2 * UM_PANEL, mm + 3 * UM_PANEL, offK, offK, kr, 32);
            }
            umma::fence_proxy_async_smem();     // generic-proxy writes -> tensor-core reads
            __syncwarp();
            if (lane == 0) {
                tma::mbar_arrive(&raw_empty[rs]);
                tma::mbar_arrive(&mma_full[ms]);
            }
            if (t == 0) trace_mark(P, 2, pi);
            ++pi;
            if (++rs == TG_RAW) { rs = 0; rph ^= 1u; }
            if (++ms == TG_MMA) { ms = 0; mph ^= 1u; }
            if (MODE == UMMA_TN && c.p + 1 == c.KP) {
                // bias gradient: column sums of dZ over this row chunk (last slot, first column tile);
                // thread t owns columns 4*(t&31)..+3 of every float4 it split
                const bool do_db = P.db && (c.s == P.rg.ks[c.t] - 1) && c.c0 == 0;
                if (do_db) {
                    const int j = t & 31;
                    atomicAdd(&dbred[4 * j + 0], cs.x);
                    atomicAdd(&dbred[4 * j + 1], cs.y);
                    atomicAdd(&dbred[4 * j + 2], cs.z);
                    atomicAdd(&dbred[4 * j + 3], cs.w);
                    tma::named_sync(1, TG_SPLIT);
                    if (t < 128 && c.n0 + t < P.N) atomicAdd(P.db + c.n0 + t, dbred[t]);
                    tma::named_sync(1, TG_SPLIT);
                    if (t < 128) dbred[t] = 0.f;
                }
                cs = make_float4(0.f, 0.f, 0.f, 0.f);
            }
            advance(c);
        }
    } else {
        // ------------------------------------------------------------- epilogue
        const int q = warp & 3;                 // TMEM lane quarter of this warp
        const int r = q * 32 + lane;            // tile row (NN/NT) or dW row k (TN)
        int as = 0, ei = 0;
        uint32_t aph = 0;
        if (q == 0 && lane == 0) trace_mark(P, 3, TG_TRACE - 1);
        while (c.tile < total) {
            if (P.dbg & 8) tma::mbar_wait_sleep(&acc_full[as], aph);
            else tma::mbar_wait_k(&acc_full[as], aph, P.dbg & 512);
            umma::tc_fence_after();
            const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(as * 128);
#pragma unroll 1
            for (int cc = 0; cc < 4; ++cc) {
                const int col = cc * 32;
                float v[32];
                umma::tmem_ld32(tbase + (uint32_t)col, v);
                if (MODE == UMMA_NN) {
                    const int64_t row = c.row0 + r;
                    if (row < c.rlim) {
                        float* out = P.C + row * P.ldc;
                        const bool vec = ((P.ldc & 3) == 0) && ((reinterpret_cast<uintptr_t>(P.C) & 15) == 0);
                        const bool split = P.ksplit > 1;
#pragma unroll
                        for (int e = 0; e < 32; e += 4) {
                            const int n = c.n0 + col + e;
                            float x[4];
#pragma unroll
                            for (int u = 0; u < 4; ++u) {
                                const bool add_b = P.bias && n + u < P.N && (!split || c.split == 0);
                                x[u] = v[e + u] + (add_b ? __ldg(P.bias + n + u) : 0.f);
                                if (P.relu && !split) x[u] = fmaxf(x[u], 0.f);
                            }
                            if (vec && n + 3 < P.N) {
                                if (split) red_add_f4(out + n, make_float4(x[0], x[1], x[2], x[3]));
                                else *reinterpret_cast<float4*>(out + n) = make_float4(x[0], x[1], x[2], x[3]);
                            } else {
                                for (int u = 0; u < 4; ++u)
                                    if (n + u < P.N) {
                                        if (split) atomicAdd(out + n + u, x[u]);
                                        else out[n + u] = x[u];
                                    }
                            }
                        }
                    }
                } else if (MODE == UMMA_NT) {
                    const int64_t row = c.row0 + r;
                    if (row < c.rlim) {
                        float* out = P.C + row * P.ldc + (int64_t)c.s * P.d_in;
                        const bool vec = ((P.ldc & 3) == 0) && ((P.d_in & 3) == 0) &&
                                         ((reinterpret_cast<uintptr_t>(P.C) & 15) == 0);
#pragma unroll
                        for (int e = 0; e < 32; e += 4) {
                            const int k = c.c0 + col + e;
                            const float4 x = make_float4(v[e], v[e + 1], v[e + 2], v[e + 3]);
                            if (vec && k + 3 < P.d_in) {
                                if (P.ksplit > 1) red_add_f4(out + k, x);
                                else *reinterpret_cast<float4*>(out + k) = x;
                            } else {
                                for (int u = 0; u < 4; ++u)
                                    if (k + u < P.d_in) {
                                        if (P.ksplit > 1) atomicAdd(out + k + u, v[e + u]);
                                        else out[k + u] = v[e + u];
                                    }
                            }
                        }
                    }
                } else {
                    const int k = c.c0 + r;
                    if (k < P.d_in) {
                        float* out = P.C + (int64_t)P.rg.slot_w[c.t][c.s] * P.bslot + (int64_t)k * P.ldc;
                        const bool vec = ((P.ldc & 3) == 0) && ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
#pragma unroll
                        for (int e = 0; e < 32; e += 4) {
                            const int n = c.n0 + col + e;
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
            umma::tc_fence_before();
            __syncwarp();
            if (q == 0 && lane == 0) trace_mark(P, 3, ei++);
            if (lane == 0) tma::mbar_arrive(&acc_empty[as]);
            if (++as == 2) { as = 0; aph ^= 1u; }
            c.tile += gridDim.x;                 // next tile of this CTA (the epilogue skips panels)
            if (c.tile < total) decode_tile<MODE>(P, c.tile, nct, kct, c);
        }
    }
    umma::tc_fence_before();
    __syncthreads();
    if (warp == 1) umma::tmem_dealloc<256>(tmem);
}

// ---------------------------------------------------------------------------- host side
// 2-D fp32 tensor map over a row-major [rows][width] matrix with row stride ld (elements):
// box = {box_w, box_h}; swz128: SWIZZLE_128B (box_w = 32), else no swizzle.  Elements
// outside [0, width) x [0, rows) are zero-filled.  false if the driver entry point is missing
// or the encoding is rejected (caller falls back to the cp.async kernel).
bool encode_tmap_f32(CUtensorMap* m, const float* base, int64_t width, int64_t rows, int64_t ld, int box_w,
                     int box_h, bool swz128);

// Weight images (gsb_weight_images_register / _refresh, weights.cu): the 3xTF32 split of a
// weight tensor W [slots][K][N], hi = rna_tf32(W) and lo = rna_tf32(W - hi), both in W's own
// layout with a 16-B aligned row stride ldn = ceil4(N), kept in caller memory and refreshed once
// per step.  The TMA-everything GEMM (gemm_tma3.cuh) loads the NN / NT B operand from them.
struct WeightImage {
    const float* W;
    int32_t slots, K, N, ldn;
    float *hi, *lo;
};
const WeightImage* find_weight_image(const float* W);

// TMA pipeline when every operand satisfies TMA's alignment rules (16-B aligned bases, row
// strides multiple of 16 B), else the cp.async kernel.  a_rows / b_rows: row extents of the
// A and B matrices (A: [a_rows][lda], B: [b_rows][ldb]); a_w / b_w: their widths.
template <int MODE>
inline gsb_status launch_gemm(const char* name, UProb P, int64_t tiles_upper, int64_t a_rows, int64_t a_w,
                              int64_t b_rows, int64_t b_w, cudaStream_t s) {
    if (P.ksplit < 1) P.ksplit = 1;
    static const int dbg_knobs = getenv("GSB_GEMM_DBG") ? atoi(getenv("GSB_GEMM_DBG")) : 0;
    P.dbg = dbg_knobs;
    P.brow = (int)(P.bslot / std::max<int64_t>(P.ldb, 1));
    P.bimg = 0;
    static int use_tma = -1;
    if (use_tma < 0) {
        const char* e = getenv("GSB_GEMM");
        use_tma = (e && strcmp(e, "umma") == 0) ? 0 : 1;
    }
    const bool aligned = ((reinterpret_cast<uintptr_t>(P.A) & 15) == 0) && ((reinterpret_cast<uintptr_t>(P.B) & 15) == 0) &&
                         ((P.lda & 3) == 0) && ((P.ldb & 3) == 0) && a_rows >= 1 && b_rows >= 1 &&
                         (MODE != UMMA_TN || P.rows_per_chunk % 32 == 0) &&
                         (MODE == UMMA_TN || P.bslot % std::max<int64_t>(P.ldb, 1) == 0);
    static const bool dbg = getenv("GSB_GEMM_DEBUG") != nullptr;
    if (dbg)
        fprintf(stderr, "[gsb] %s: tma=%d aligned=%d (A %p lda %lld, B %p ldb %lld, bslot %lld)\n", name, use_tma,
                (int)aligned, (const void*)P.A, (long long)P.lda, (const void*)P.B, (long long)P.ldb,
                (long long)P.bslot);
    if (use_tma && aligned) {
        CUtensorMap ma, mb;
        const bool kA = (MODE != UMMA_TN), kB = (MODE == UMMA_NT);
        bool ok = encode_tmap_f32(&ma, P.A, a_w, a_rows, P.lda, kA ? 32 : 128, kA ? 128 : 32, kA) &&
                  encode_tmap_f32(&mb, P.B, b_w, b_rows, P.ldb, kB ? 32 : 128, kB ? 128 : 32, kB);
        if (ok) {
            static bool attr_set = false;
            if (!attr_set) {
                GSB_CUDA(cudaFuncSetAttribute(tma_gemm_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              TG_SMEM));
                attr_set = true;
            }
            const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles_upper * P.ksplit, kNumSMs));
            GSB_LAUNCH(name, tma_gemm_kernel<MODE>, grid, TG_THREADS, TG_SMEM, s, ma, mb, mb, P);
            return GSB_OK;
        }
        if (dbg) fprintf(stderr, "[gsb] %s: tensor map encoding failed\n", name);
    }
    return launch_umma<MODE>(name, P, tiles_upper, s);
}

}  // namespace gsb
