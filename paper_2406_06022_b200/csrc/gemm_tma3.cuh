// gemm_tma3.cuh -- the grouped RGCN GEMMs (modes NN / NT / TN, tile schedule and epilogues of
// gemm_umma.cuh) with every operand moved by TMA straight into its UMMA layout.
//
// 3xTF32 without a hi copy: kind::tf32 reads a 32-bit operand as its truncation to tf32 (low
// 13 mantissa bits ignored; measured bit-exact, scripts/probe_tf32.cu (a)), so the raw fp32
// panel TMA delivers IS the hi operand; the splitters only write lo = x - trunc(x) (exact in
// fp32) at the same offsets.  D += A_lo B_hi + A_hi B_lo + A_hi B_hi.
//
// Layouts (both probed, scripts/probe_tf32.cu (b), (d)):
//   K-major  operand panel 128 x 32: TMA SWIZZLE_128B box {32, 128}; desc LBO 16 / SBO 1024,
//            k-step advance 32 B.
//   MN-major operand panel 32 (k) x 128 (mn): 4 TMA boxes {32 mn, 32 k} with
//            SWIZZLE_128B_ATOM_32B at 4096 B apart; desc (SWIZZLE_128B_BASE32B) LBO 4096 (MN atom
//            stride) / SBO 512 (4-row K group stride), k-step advance 1024 B.
//
// Epilogue through shared memory: the accumulator (TMEM) is read 32 columns at a time, written
// to a SWIZZLE_128B staging tile and stored by one TMA store (or TMA reduce-add for split-K and
// the weight gradients), so the global writes are bulk and coalesced instead of one 16-B store
// per lane per row.  Tiles cut by a group end (rows of the next group follow) use per-thread
// stores.
//
//   warp 0      TMA producer (lane 0)
//   warp 1      TMEM owner + MMA issuer (lane 0)
//   warps 2..   lo splitters (T3_SPLIT_WARPS)
//   last 4      epilogue
#pragma once
#include <cuda.h>

#include "gemm_tma.cuh"

namespace gsb {

namespace tma {
__device__ __forceinline__ void store_2d(const CUtensorMap* map, int32_t c0, int32_t c1, uint32_t src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(src)
                 : "memory");
}
__device__ __forceinline__ void redadd_2d(const CUtensorMap* map, int32_t c0, int32_t c1, uint32_t src) {
    asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(src)
                 : "memory");
}
__device__ __forceinline__ void store_3d(const CUtensorMap* map, int32_t c0, int32_t c1, int32_t c2, uint32_t src) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(c2), "r"(src)
                 : "memory");
}
__device__ __forceinline__ void redadd_3d(const CUtensorMap* map, int32_t c0, int32_t c1, int32_t c2, uint32_t src) {
    asm volatile(
        "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
            reinterpret_cast<uint64_t>(map)),
        "r"(c0), "r"(c1), "r"(c2), "r"(src)
        : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
// L2 prefetch of one TMA box (no shared-memory destination, no completion)
__device__ __forceinline__ void prefetch_2d(const CUtensorMap* map, int32_t c0, int32_t c1) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1)
                 : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
}  // namespace tma

#ifndef GSB_T3_SPLIT_WARPS
#define GSB_T3_SPLIT_WARPS 4
#endif
constexpr int T3_SPLIT_WARPS = GSB_T3_SPLIT_WARPS;
constexpr int T3_SPLIT = 32 * T3_SPLIT_WARPS;
constexpr int T3_EPI_WARP0 = 2 + T3_SPLIT_WARPS;
constexpr int T3_THREADS = 32 * (T3_EPI_WARP0 + 4);
constexpr int T3_PER = 1024 / T3_SPLIT;            // float4 of one operand panel per splitter thread
constexpr int T3_STAGE = 4 * UM_PANEL;             // A raw(hi), A lo, B raw(hi), B lo
constexpr int T3_OUT = UM_PANEL;                   // one 128 x 32 fp32 epilogue staging tile
constexpr int t3_smem(int stages) { return stages * T3_STAGE + 2 * T3_OUT + 1024; }

// lo = x - trunc_tf32(x) (exact in fp32; the tf32 hi the tensor core reads from the raw value),
// rounded to tf32 to nearest here: the tensor core would truncate it, and truncation errors all
// carry the sign of x (a bias that does not average out in long sums)
__device__ __forceinline__ float lo_of(float x) {
    const float r = x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
    return __uint_as_float(umma::rna_tf32_bits(__float_as_uint(r)));
}

// desc of an MN-major panel as TMA ATOM_32B lays it out (4 boxes {32 mn, 32 k} 4096 B apart)
__device__ __forceinline__ uint64_t desc_mn_tma(uint32_t addr) { return umma::desc_encode(addr, 4096, 512, 1); }

// per-thread float4 byte offsets in an operand panel.  K-major: linear (conflict-free).
// MN-major: thread t owns the 4 columns mn = 4*(t&31) .. +3 (atom j = (t&31)>>3, 32-B chunk
// lc = (t>>1)&3, half = t&1) of K rows kk = (t>>5) + T3_SPLIT_WARPS*i, so its TN column sums
// stay in registers; the swizzled chunk is lc ^ (kk&3).
struct T3Off {
    uint32_t k[T3_PER];
    uint32_t m[T3_PER];
    int kk[T3_PER];
};
__device__ __forceinline__ T3Off t3_offsets(int t) {
    T3Off o;
    const int l = t & 31, j = l >> 3, lc = (l >> 1) & 3, half = l & 1;
#pragma unroll
    for (int i = 0; i < T3_PER; ++i) {
        o.k[i] = 16u * (uint32_t)(t + T3_SPLIT * i);
        const int kk = (t >> 5) + T3_SPLIT_WARPS * i;
        o.kk[i] = kk;
        o.m[i] = (uint32_t)(j * 4096 + kk * 128 + ((lc ^ (kk & 3)) << 5) + (half << 4));
    }
    return o;
}

// lo of one operand panel; ZERO: K rows kk >= klim are zeroed in raw and lo (TN chunk ends);
// CS: column sums of the (zeroed) values, per thread (TN bias gradient).
// HI: also round the hi operand to nearest in place (hi = rna_tf32(x), lo = rna_tf32(x - hi))
// for ONE of the two operands: with both his truncated the dropped lo_A lo_B term has the sign
// of every product (both residuals carry the sign of their x) and accumulates like the result
// itself; one round-to-nearest residual makes it zero-mean (the 3xTF32 accuracy of an rna split)
template <bool MN, bool ZERO, bool CS, bool HI>
__device__ __forceinline__ void t3_split(uint32_t raw, uint32_t lo, const T3Off& o, int klim, double4& cs) {
    float4 v[T3_PER];
#pragma unroll
    for (int i = 0; i < T3_PER; ++i) v[i] = lds128(raw + (MN ? o.m[i] : o.k[i]));
#pragma unroll
    for (int i = 0; i < T3_PER; ++i) {
        const uint32_t off = MN ? o.m[i] : o.k[i];
        if (ZERO && o.kk[i] >= klim) {
            v[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (!HI) sts128(raw + off, 0u, 0u, 0u, 0u);
        }
        if (CS) { cs.x += v[i].x; cs.y += v[i].y; cs.z += v[i].z; cs.w += v[i].w; }   // fp64: exact-ish sums
        if (HI) {
            uint32_t h0, h1, h2, h3, l0, l1, l2, l3;
            umma::split_tf32(v[i].x, h0, l0);
            umma::split_tf32(v[i].y, h1, l1);
            umma::split_tf32(v[i].z, h2, l2);
            umma::split_tf32(v[i].w, h3, l3);
            sts128(raw + off, h0, h1, h2, h3);
            sts128(lo + off, l0, l1, l2, l3);
        } else {
            sts128(lo + off, __float_as_uint(lo_of(v[i].x)), __float_as_uint(lo_of(v[i].y)),
                   __float_as_uint(lo_of(v[i].z)), __float_as_uint(lo_of(v[i].w)));
        }
    }
}

// Per-thread global stores of one 32-column chunk (tiles the TMA store cannot take): the
// gemm_tma.cuh epilogue.
template <int MODE>
__device__ __forceinline__ void t3_epi_direct(const UProb& P, const UCursor& c, int r, int col, const float (&v)[32]) {
    if (MODE == UMMA_NN) {
        const int64_t row = c.row0 + r;
        if (row >= c.rlim) return;
        float* out = P.C + row * P.ldc;
        const bool split = P.ksplit > 1;
#pragma unroll
        for (int e = 0; e < 32; ++e) {
            const int n = c.n0 + col + e;
            if (n >= P.N) break;
            float x = v[e] + ((P.bias && (!split || c.split == 0)) ? __ldg(P.bias + n) : 0.f);
            if (P.relu && !split) x = fmaxf(x, 0.f);
            if (split) atomicAdd(out + n, x);
            else out[n] = x;
        }
    } else if (MODE == UMMA_NT) {
        const int64_t row = c.row0 + r;
        if (row >= c.rlim) return;
        float* out = P.C + row * P.ldc + (int64_t)c.s * P.d_in;
#pragma unroll
        for (int e = 0; e < 32; ++e) {
            const int k = c.c0 + col + e;
            if (k >= P.d_in) break;
            if (P.ksplit > 1) atomicAdd(out + k, v[e]);
            else out[k] = v[e];
        }
    } else {                  // TN with a C the TMA cannot address (e.g. a 349-column dWc)
        const int k = c.c0 + r;
        if (k >= P.d_in) return;
        float* out = P.C + (int64_t)P.rg.slot_w[c.t][c.s] * P.bslot + (int64_t)k * P.ldc;
#pragma unroll
        for (int e = 0; e < 32; ++e) {
            const int n = c.n0 + col + e;
            if (n >= P.N) break;
            atomicAdd(out + n, v[e]);
        }
    }
}

// maps: A, B operands; C output (NN: 2-D [rows][N]; NT: 3-D {d_in, slots, rows}; TN: 3-D
// {N, d_in, slots}), box 32 x 128 SWIZZLE_128B
// P.bimg: the NN / NT B operand comes pre-split from weight images (mapB = hi, mapB2 = lo,
// both rna; weights.cu), so the splitters only write A's lo
template <int MODE, int T3_STAGES>
__global__ void __launch_bounds__(T3_THREADS, 1) tma3_gemm_kernel(const __grid_constant__ CUtensorMap mapA,
                                                                   const __grid_constant__ CUtensorMap mapB,
                                                                   const __grid_constant__ CUtensorMap mapB2,
                                                                   const __grid_constant__ CUtensorMap mapC, UProb P) {
    if (threadIdx.x == 0) trace_mark(P, 0, TG_TRACE - 2);
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* ring = smem;
    uint8_t* outbuf = smem + T3_STAGES * T3_STAGE;
    __shared__ __align__(8) uint64_t full[T3_STAGES], split_done[T3_STAGES], empty[T3_STAGES];
    __shared__ __align__(8) uint64_t acc_full[2], acc_empty[2];
    __shared__ uint32_t tmem_sh;
    __shared__ double dbred[128];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    constexpr bool A_MN = (MODE == UMMA_TN);
    constexpr bool B_MN = (MODE != UMMA_NT);

    if (tid == 0) {
        for (int s = 0; s < T3_STAGES; ++s) {
            umma::mbar_init(&full[s], 1);
            umma::mbar_init(&split_done[s], T3_SPLIT_WARPS);
            umma::mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            umma::mbar_init(&acc_full[s], 1);
            umma::mbar_init(&acc_empty[s], 4);
        }
        umma::fence_barrier_init();
        tma::prefetch_map(&mapA);
        tma::prefetch_map(&mapB);
        if (P.bimg) tma::prefetch_map(&mapB2);
        tma::prefetch_map(&mapC);
    }
    if (tid < 128) dbred[tid] = 0.0;
    if (warp == 1) umma::tmem_alloc<256>(&tmem_sh);
    umma::tc_fence_before();
    __syncthreads();
    umma::tc_fence_after();
    const uint32_t tmem = tmem_sh;
    // with PDL (GSB_PDL=1) the setup above overlaps the predecessor's tail; nothing it wrote
    // (row-group sizes, operands) is read before this point
    GSB_PDL_ENTRY();

    const int nct = (P.N + 127) / 128;
    const int kct = (P.d_in + 127) / 128;
    const int64_t total = (P.dbg & 64) ? 0 : total_tiles<MODE>(P, nct, kct);

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
            int st = 0, pi = 0;
            uint32_t ph = 0;
            // L2 prefetch of the HBM-streamed operands P.pf panels ahead of the loads (A of NN / NT
            // -- Acat, dZ -- and both TN operands), so the ring's TMA loads hit L2
            UCursor pc = c;
            for (int k = 0; k < P.pf && pc.tile < total; ++k) advance(pc);
            while (c.tile < total) {
                if (P.pf > 0 && pc.tile < total) {
                    if (MODE == UMMA_NN) {
                        const int per = P.d_in / 32, sp = pc.p / per, kk = (pc.p - sp * per) * 32;
                        tma::prefetch_2d(&mapA, sp * P.d_in + kk, (int32_t)pc.row0);
                    } else if (MODE == UMMA_NT) {
                        tma::prefetch_2d(&mapA, pc.p * 32, (int32_t)pc.row0);
                    } else {
                        const int32_t rb = (int32_t)(pc.row0 + (int64_t)pc.p * 32);
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            tma::prefetch_2d(&mapA, pc.s * P.d_in + pc.c0 + 32 * j, rb);
                            tma::prefetch_2d(&mapB, pc.n0 + 32 * j, rb);
                        }
                    }
                    advance(pc);
                }
                if (P.dbg & 2048) trace_mark(P, 0, 3 * pi);
                tma::mbar_wait_k(&empty[st], ph ^ 1u, P.dbg & 512);
                if (P.dbg & 2048) trace_mark(P, 0, 3 * pi + 1);
                const uint32_t a = umma::smem_u32(ring + st * T3_STAGE), b = a + 2 * UM_PANEL;
                if (P.dbg & 4) {
                    tma::mbar_arrive(&full[st]);    // A/B knob: no loads
                } else if (MODE == UMMA_NN) {
                    tma::mbar_expect_tx(&full[st], (P.bimg ? 3 : 2) * UM_PANEL);
                    const int per = P.d_in / 32;
                    const int sp = c.p / per;
                    const int kk = (c.p - sp * per) * 32;
                    tma::load_2d(a, &mapA, sp * P.d_in + kk, (int32_t)c.row0, &full[st]);
                    const int32_t wrow = P.rg.slot_w[c.t][sp] * P.brow + kk;
#pragma unroll
                    for (int j = 0; j < 4; ++j) tma::load_2d(b + j * 4096, &mapB, c.n0 + 32 * j, wrow, &full[st]);
                    if (P.bimg) {
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            tma::load_2d(b + UM_PANEL + j * 4096, &mapB2, c.n0 + 32 * j, wrow, &full[st]);
                    }
                } else if (MODE == UMMA_NT) {
                    tma::mbar_expect_tx(&full[st], (P.bimg ? 3 : 2) * UM_PANEL);
                    tma::load_2d(a, &mapA, c.p * 32, (int32_t)c.row0, &full[st]);
                    const int32_t wrow = P.rg.slot_w[c.t][c.s] * P.brow + c.c0;
                    tma::load_2d(b, &mapB, c.p * 32, wrow, &full[st]);
                    if (P.bimg) tma::load_2d(b + UM_PANEL, &mapB2, c.p * 32, wrow, &full[st]);
                } else {
                    tma::mbar_expect_tx(&full[st], 2 * UM_PANEL);
                    const int32_t rb = (int32_t)(c.row0 + (int64_t)c.p * 32);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        tma::load_2d(a + j * 4096, &mapA, c.s * P.d_in + c.c0 + 32 * j, rb, &full[st]);
                        tma::load_2d(b + j * 4096, &mapB, c.n0 + 32 * j, rb, &full[st]);
                    }
                }
                trace_mark(P, 0, (P.dbg & 2048) ? 3 * pi + 2 : pi);
                ++pi;
                if (++st == T3_STAGES) { st = 0; ph ^= 1u; }
                advance(c);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------- MMA issuer
        if (lane == 0) {
            const uint32_t IDESC = umma::idesc_tf32(128, A_MN, B_MN);
            int st = 0, as = 0, pi = 0;
            uint32_t ph = 0, aph = 0;
            while (c.tile < total) {
                if (c.p == c.p0) {
                    tma::mbar_wait_k(&acc_empty[as], aph ^ 1u, P.dbg & 512);
                    umma::tc_fence_after();
                }
                tma::mbar_wait_k(&split_done[st], ph, P.dbg & 512);
                umma::tc_fence_after();
                const uint32_t a_hi = umma::smem_u32(ring + st * T3_STAGE), a_lo = a_hi + UM_PANEL;
                const uint32_t b_hi = a_hi + 2 * UM_PANEL, b_lo = a_hi + 3 * UM_PANEL;
                const uint32_t d = tmem + (uint32_t)(as * 128);
#pragma unroll
                for (int ks = 0; ks < ((P.dbg & 2) ? 0 : 4); ++ks) {
                    const uint32_t oa = A_MN ? ks * 1024u : ks * 32u;
                    const uint32_t ob = B_MN ? ks * 1024u : ks * 32u;
                    const uint64_t dah = A_MN ? desc_mn_tma(a_hi + oa) : umma::desc_kmajor(a_hi + oa);
                    const uint64_t dal = A_MN ? desc_mn_tma(a_lo + oa) : umma::desc_kmajor(a_lo + oa);
                    const uint64_t dbh = B_MN ? desc_mn_tma(b_hi + ob) : umma::desc_kmajor(b_hi + ob);
                    const uint64_t dbl = B_MN ? desc_mn_tma(b_lo + ob) : umma::desc_kmajor(b_lo + ob);
                    umma::mma_tf32(d, dal, dbh, IDESC, (c.p > c.p0 || ks > 0) ? 1u : 0u);
                    umma::mma_tf32(d, dah, dbl, IDESC, 1u);
                    umma::mma_tf32(d, dah, dbh, IDESC, 1u);
                }
                trace_mark(P, 1, pi++);
                umma::mma_commit(&empty[st]);
                if (++st == T3_STAGES) { st = 0; ph ^= 1u; }
                if (c.p + 1 == c.KP) {
                    umma::mma_commit(&acc_full[as]);
                    if (++as == 2) { as = 0; aph ^= 1u; }
                }
                advance(c);
            }
        }
    } else if (warp < T3_EPI_WARP0) {
        // ------------------------------------------------------------- lo splitters
        const int t = tid - 64;
        const T3Off o = t3_offsets(t);
        int st = 0, pi = 0;
        uint32_t ph = 0;
        double4 cs = make_double4(0.0, 0.0, 0.0, 0.0);
        while (c.tile < total) {
            tma::mbar_wait_k(&full[st], ph, P.dbg & 512);
            const uint32_t a = umma::smem_u32(ring + st * T3_STAGE), b = a + 2 * UM_PANEL;
            if (P.dbg & 1) {
            } else if (MODE == UMMA_TN) {
                const int64_t rb = c.row0 + (int64_t)c.p * 32;
                const int klim = (int)min((int64_t)32, c.rlim - rb);
                if (klim < 32) {
                    t3_split<true, true, false, false>(a, a + UM_PANEL, o, klim, cs);
                    t3_split<true, true, true, true>(b, b + UM_PANEL, o, klim, cs);
                } else {
                    t3_split<true, false, false, false>(a, a + UM_PANEL, o, 32, cs);
                    t3_split<true, false, true, true>(b, b + UM_PANEL, o, 32, cs);
                }
            } else if (MODE == UMMA_NN) {
                t3_split<false, false, false, false>(a, a + UM_PANEL, o, 32, cs);
                if (!P.bimg) t3_split<true, false, false, true>(b, b + UM_PANEL, o, 32, cs);
            } else {
                t3_split<false, false, false, false>(a, a + UM_PANEL, o, 32, cs);
                if (!P.bimg) t3_split<false, false, false, true>(b, b + UM_PANEL, o, 32, cs);
            }
            umma::fence_proxy_async_smem();     // generic-proxy writes -> tensor-core reads
            __syncwarp();
            if (lane == 0) tma::mbar_arrive(&split_done[st]);
            if (t == 0) trace_mark(P, 2, pi);
            ++pi;
            if (++st == T3_STAGES) { st = 0; ph ^= 1u; }
            if (MODE == UMMA_TN && c.p + 1 == c.KP) {
                // bias gradient: column sums of dZ over this row chunk (last slot, first k tile);
                // thread t owns columns 4*(t&31)..+3
                const bool do_db = P.db && (c.s == P.rg.ks[c.t] - 1) && c.c0 == 0;
                if (do_db) {
                    const int j = 4 * (t & 31);
                    atomicAdd(&dbred[j + 0], cs.x);
                    atomicAdd(&dbred[j + 1], cs.y);
                    atomicAdd(&dbred[j + 2], cs.z);
                    atomicAdd(&dbred[j + 3], cs.w);
                    tma::named_sync(1, T3_SPLIT);
                    if (t < 128 && c.n0 + t < P.N) atomicAdd(P.db + c.n0 + t, (float)dbred[t]);
                    tma::named_sync(1, T3_SPLIT);
                    if (t < 128) dbred[t] = 0.0;
                }
                cs = make_double4(0.0, 0.0, 0.0, 0.0);
            }
            advance(c);
        }
    } else {
        // ------------------------------------------------------------- epilogue
        const int q = warp & 3;                 // TMEM lane quarter of this warp
        const int r = q * 32 + lane;            // tile row (NN/NT) or dW row k (TN)
        const int et = tid - 32 * T3_EPI_WARP0; // 0..127
        int as = 0, ei = 0, ob = 0;
        uint32_t aph = 0;
        while (c.tile < total) {
            tma::mbar_wait_k(&acc_full[as], aph, P.dbg & 512);
            umma::tc_fence_after();
            if (et == 0) trace_mark(P, 3, 8 * ei);
            const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(as * 128);
            const bool split = (MODE == UMMA_TN) || P.ksplit > 1;
            // a tile cut by its group end (next group's rows follow) cannot take a box store
            const bool direct = P.cdirect || ((MODE != UMMA_TN) && (c.row0 + 128 > c.rlim));
#pragma unroll 1
            for (int cc = 0; cc < 4; ++cc) {
                const int col = cc * 32;
                const int lim = (MODE == UMMA_NT) ? P.d_in - c.c0 : P.N - c.n0;
                if (col >= lim) break;          // uniform: chunk past the output width
                float v[32];
                umma::tmem_ld32(tbase + (uint32_t)col, v);
                const bool tr = (P.dbg & 4096) && et == 0 && ei == 0 && cc == 0;
                if (tr) trace_mark(P, 2, 32);
                if (P.dbg & 8) continue;        // A/B knob: no stores
                if (direct) {
                    t3_epi_direct<MODE>(P, c, r, col, v);
                    continue;
                }
                if (MODE == UMMA_NN) {
                    // bias (uniform per chunk: same 32 values for every row) and relu
                    if (P.bias && (!split || c.split == 0)) {
                        const float* bp = P.bias + c.n0 + col;
                        if (c.n0 + col + 32 <= P.N && (reinterpret_cast<uintptr_t>(bp) & 15) == 0) {
#pragma unroll
                            for (int e = 0; e < 32; e += 4) {
                                const float4 b4 = __ldg(reinterpret_cast<const float4*>(bp + e));
                                v[e] += b4.x; v[e + 1] += b4.y; v[e + 2] += b4.z; v[e + 3] += b4.w;
                            }
                        } else {
                            const int nv = P.N - c.n0 - col;
#pragma unroll
                            for (int e = 0; e < 32; ++e) v[e] += (e < nv) ? __ldg(bp + e) : 0.f;
                        }
                    }
                    if (P.relu && !split) {
#pragma unroll
                        for (int e = 0; e < 32; ++e) v[e] = fmaxf(v[e], 0.f);
                    }
                }
                if (tr) trace_mark(P, 2, 33);
                const uint32_t buf = umma::smem_u32(outbuf + ob * T3_OUT);
                if (et == 0) tma::bulk_wait_read<1>();   // the store that used this buffer has read it
                if (tr) trace_mark(P, 2, 34);
                tma::named_sync(2, 128);
                if (tr) trace_mark(P, 2, 35);
#pragma unroll
                for (int e = 0; e < 32; e += 4)
                    sts128(buf + umma::kmajor_off(r, e), __float_as_uint(v[e]), __float_as_uint(v[e + 1]),
                           __float_as_uint(v[e + 2]), __float_as_uint(v[e + 3]));
                if (tr) trace_mark(P, 2, 36);
                umma::fence_proxy_async_smem();
                if (tr) trace_mark(P, 2, 37);
                tma::named_sync(2, 128);
                if (tr) trace_mark(P, 2, 38);
                if (et == 0) {
                    if (MODE == UMMA_NN) {
                        if (split) tma::redadd_2d(&mapC, c.n0 + col, (int32_t)c.row0, buf);
                        else tma::store_2d(&mapC, c.n0 + col, (int32_t)c.row0, buf);
                    } else if (MODE == UMMA_NT) {
                        if (split) tma::redadd_3d(&mapC, c.c0 + col, c.s, (int32_t)c.row0, buf);
                        else tma::store_3d(&mapC, c.c0 + col, c.s, (int32_t)c.row0, buf);
                    } else {
                        tma::redadd_3d(&mapC, c.n0 + col, c.c0, P.rg.slot_w[c.t][c.s], buf);
                    }
                    tma::bulk_commit();
                    trace_mark(P, 3, 8 * ei + 1 + cc);
                }
                ob ^= 1;
            }
            umma::tc_fence_before();
            __syncwarp();
            if (et == 0) trace_mark(P, 3, 8 * ei + 5);
            ++ei;
            if (lane == 0) tma::mbar_arrive(&acc_empty[as]);
            if (++as == 2) { as = 0; aph ^= 1u; }
            c.tile += gridDim.x;
            if (c.tile < total) decode_tile<MODE>(P, c.tile, nct, kct, c);
        }
        if (et == 0) {
            tma::bulk_wait_all();
            trace_mark(P, 3, TG_TRACE - 2);
        }
    }
    umma::tc_fence_before();
    __syncthreads();
    if (warp == 1) umma::tmem_dealloc<256>(tmem);
}

// ---------------------------------------------------------------------------- host side
// general fp32 tensor map: rank 2 or 3, dims / strides (elements, innermost first; strides of
// dims 1..rank-1), box, swizzle (CUtensorMapSwizzle).  false if rejected.
bool encode_tmap_nd(CUtensorMap* m, const float* base, int rank, const int64_t* dims, const int64_t* strides,
                    const int* box, int swizzle);

// TMA-everything pipeline.  *launched = false (nothing enqueued) if a tensor map cannot be
// encoded; the caller then falls back to the other kernels.  c_rows: rows of C (NN / NT);
// c_slots: TN: weight slots of C (dW), NT: column slots per row of C (dacat).
template <int MODE>
inline gsb_status launch_gemm3(const char* name, UProb P, int64_t tiles_upper, int64_t a_rows, int64_t a_w,
                               int64_t b_rows, int64_t b_w, int64_t c_rows, int64_t c_slots, cudaStream_t s,
                               bool* launched, const WeightImage* wi = nullptr) {
    *launched = false;
    CUtensorMap ma, mb, mb2, mc;
    const int SW128 = CU_TENSOR_MAP_SWIZZLE_128B, SW32 = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
    bool ok;
    if (MODE == UMMA_NN) {
        const int64_t da[2] = {a_w, a_rows}, sa[1] = {P.lda};
        const int64_t db[2] = {b_w, b_rows}, sb[1] = {P.ldb};
        const int64_t dc[2] = {P.N, c_rows}, sc[1] = {P.ldc};
        const int ba[2] = {32, 128}, bb[2] = {32, 32}, bc[2] = {32, 128};
        ok = encode_tmap_nd(&ma, P.A, 2, da, sa, ba, SW128) &&
             (P.cdirect || encode_tmap_nd(&mc, P.C, 2, dc, sc, bc, SW128));
        if (wi) {
            const int64_t di[2] = {wi->N, (int64_t)wi->slots * wi->K}, si[1] = {wi->ldn};
            ok = ok && encode_tmap_nd(&mb, wi->hi, 2, di, si, bb, SW32) && encode_tmap_nd(&mb2, wi->lo, 2, di, si, bb, SW32);
        } else {
            ok = ok && encode_tmap_nd(&mb, P.B, 2, db, sb, bb, SW32);
        }
    } else if (MODE == UMMA_NT) {
        const int64_t da[2] = {a_w, a_rows}, sa[1] = {P.lda};
        const int64_t db[2] = {b_w, b_rows}, sb[1] = {P.ldb};
        const int64_t dc[3] = {P.d_in, c_slots, c_rows}, sc[2] = {P.d_in, P.ldc};
        const int ba[2] = {32, 128}, bb[2] = {32, 128}, bc[3] = {32, 1, 128};
        ok = encode_tmap_nd(&ma, P.A, 2, da, sa, ba, SW128) &&
             (P.cdirect || encode_tmap_nd(&mc, P.C, 3, dc, sc, bc, SW128));
        if (wi) {
            const int64_t di[2] = {wi->N, (int64_t)wi->slots * wi->K}, si[1] = {wi->ldn};
            ok = ok && encode_tmap_nd(&mb, wi->hi, 2, di, si, bb, SW128) &&
                 encode_tmap_nd(&mb2, wi->lo, 2, di, si, bb, SW128);
        } else {
            ok = ok && encode_tmap_nd(&mb, P.B, 2, db, sb, bb, SW128);
        }
    } else {
        const int64_t da[2] = {a_w, a_rows}, sa[1] = {P.lda};
        const int64_t db[2] = {b_w, b_rows}, sb[1] = {P.ldb};
        const int64_t dc[3] = {P.N, P.d_in, c_slots},
                      sc[2] = {P.ldc, P.bslot > 0 ? P.bslot : (int64_t)P.d_in * P.ldc};
        const int ba[2] = {32, 32}, bb[2] = {32, 32}, bc[3] = {32, 128, 1};
        ok = encode_tmap_nd(&ma, P.A, 2, da, sa, ba, SW32) && encode_tmap_nd(&mb, P.B, 2, db, sb, bb, SW32) &&
             (P.cdirect || encode_tmap_nd(&mc, P.C, 3, dc, sc, bc, SW128));
    }
    if (!ok) return GSB_OK;
    if (P.cdirect) mc = ma;      // C not TMA-addressable: per-thread stores, map unused
    P.bimg = wi ? 1 : 0;
    if (!wi) mb2 = mb;
    // operand ring depth: 3 stages (225 KB, one CTA per SM) or 2 (161 KB: leaves room for
    // the concurrently running sample-phase kernels on the same SM); GSB_T3_STAGES
    static const int stages = (getenv("GSB_T3_STAGES") && atoi(getenv("GSB_T3_STAGES")) == 2) ? 2 : 3;
    static bool attr_set = false;
    if (!attr_set) {
        GSB_CUDA(cudaFuncSetAttribute(tma3_gemm_kernel<MODE, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      t3_smem(2)));
        GSB_CUDA(cudaFuncSetAttribute(tma3_gemm_kernel<MODE, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      t3_smem(3)));
        attr_set = true;
    }
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles_upper * P.ksplit, kNumSMs));
    if (stages == 2)
        GSB_LAUNCH(name, (tma3_gemm_kernel<MODE, 2>), grid, T3_THREADS, t3_smem(2), s, ma, mb, mb2, mc, P);
    else
        GSB_LAUNCH(name, (tma3_gemm_kernel<MODE, 3>), grid, T3_THREADS, t3_smem(3), s, ma, mb, mb2, mc, P);
    *launched = true;
    return GSB_OK;
}

// GEMM dispatch: the TMA-everything kernel above when every operand suits TMA (16-B aligned
// bases, row strides multiple of 16 B), else launch_gemm (gemm_tma.cuh: the split-in-smem TMA
// kernel or the cp.async kernel).  GSB_GEMM=tma2 | umma selects those for A/B runs.
inline int gemm_version() {
    static int ver = -1;
    if (ver < 0) {
        const char* e = getenv("GSB_GEMM");
        ver = (e && (strcmp(e, "tma2") == 0 || strcmp(e, "umma") == 0)) ? 2 : 3;
    }
    return ver;
}

template <int MODE>
inline gsb_status launch_gemm_v(const char* name, UProb P, int64_t tiles_upper, int64_t a_rows, int64_t a_w,
                                int64_t b_rows, int64_t b_w, cudaStream_t s) {
    const int ver = gemm_version();
    if (ver == 3) {
        UProb Q = P;
        if (Q.ksplit < 1) Q.ksplit = 1;
        static const int dbg_knobs = getenv("GSB_GEMM_DBG") ? atoi(getenv("GSB_GEMM_DBG")) : 0;
        Q.dbg = dbg_knobs;
        Q.brow = (int)(Q.bslot / std::max<int64_t>(Q.ldb, 1));
        Q.bimg = 0;
        // L2 prefetch distance (panels) of the HBM-streamed operands: opt-in, measured neutral to
        // -1 % in the step (0.2052 vs 0.2063-0.2075 ms for 2 / 4 / 8, gpurun_out/pf1)
        static const int pf = getenv("GSB_GEMM_PF") ? atoi(getenv("GSB_GEMM_PF")) : 0;
        Q.pf = pf;
        auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
        // registered weight image of the B operand (NN / NT): pre-split hi / lo, TMA'd directly
        // (also when W itself is not TMA-addressable, e.g. the 349-column decoder weight)
        static const bool no_img = getenv("GSB_NO_WIMG") != nullptr;    // A/B knob
        const WeightImage* wi = (MODE != UMMA_TN && !no_img) ? find_weight_image(Q.B) : nullptr;
        if (wi && !(wi->N == Q.N && wi->K == Q.d_in &&
                    ((int64_t)wi->K * wi->N == Q.bslot || (Q.bslot == 0 && wi->slots == 1))))
            wi = nullptr;
        const bool b_ok = wi || (al(Q.B) && (Q.ldb & 3) == 0 &&
                                 (MODE == UMMA_TN || Q.bslot % std::max<int64_t>(Q.ldb, 1) == 0));
        // C: TMA store / reduce-add when addressable, else per-thread stores / atomics
        Q.cdirect = !(al(Q.C) && (Q.ldc & 3) == 0 && (MODE != UMMA_TN || (Q.bslot & 3) == 0));
        bool ok = al(Q.A) && (Q.lda & 3) == 0 && b_ok && a_rows >= 1 && b_rows >= 1;
        int64_t c_slots = 1;
        if (MODE == UMMA_TN) {
            ok = ok && Q.rows_per_chunk % 32 == 0;
            for (int t = 0; t < Q.rg.G; ++t)
                for (int k = 0; k < Q.rg.ks[t]; ++k) c_slots = std::max<int64_t>(c_slots, Q.rg.slot_w[t][k] + 1);
        } else if (MODE == UMMA_NT) {
            c_slots = (Q.ldc % Q.d_in == 0) ? Q.ldc / Q.d_in : 1;
        }
        if (ok) {
            bool launched = false;
            const gsb_status st = launch_gemm3<MODE>(name, Q, tiles_upper, a_rows, a_w, b_rows, b_w, a_rows, c_slots, s,
                                                     &launched, wi);
            if (st != GSB_OK || launched) return st;
        }
    }
    return launch_gemm<MODE>(name, P, tiles_upper, a_rows, a_w, b_rows, b_w, s);
}

}  // namespace gsb
