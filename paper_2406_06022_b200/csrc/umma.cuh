// umma.cuh -- minimal sm_100a tcgen05 / TMEM / mbarrier wrappers (inline PTX).
//
// Operand tiles live in shared memory in the canonical SWIZZLE_128B layouts:
//   K-major  panel (128 rows x 32 tf32): row r at r*128 B, 16-B chunk c stored at chunk c ^ (r&7);
//            8-row groups 1024 B apart (SBO); one MMA (K=8 tf32 = 32 B) starts at base + ks*32.
//   MN-major panel (128 MN x 32 K), tf32 => SWIZZLE_128B_BASE32B (the only MN-major tf32 layout):
//            atoms of 32 MN (128 B) x 4 K-rows (512 B), 32-B chunk c stored at c ^ (k&3);
//            MN atoms 512 B apart (LBO), 4-row K groups 2048 B apart (SBO);
//            one MMA (K = 8 rows) starts at base + ks*4096.
// Both panels are 16 KB and must be 1024-B aligned.
#pragma once
#include <stdint.h>

namespace gsb {
namespace umma {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- descriptors -------------------------------------------------------------------
__device__ __forceinline__ uint64_t desc_encode(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= 1ull << 46;                    // descriptor version (sm_100)
    d |= (uint64_t)(layout & 7) << 61;  // 2 = SWIZZLE_128B, 1 = SWIZZLE_128B_BASE32B
    return d;
}
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t addr) { return desc_encode(addr, 16, 1024, 2); }
__device__ __forceinline__ uint64_t desc_mnmajor(uint32_t addr) { return desc_encode(addr, 512, 2048, 1); }

// kind::tf32 (a_fmt = b_fmt = TF32), fp32 accumulate, M = 128, N = n
__host__ __device__ constexpr uint32_t idesc_tf32(int n, bool a_mn, bool b_mn) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
           ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
}

// kind::f16 with bf16 A and B, fp32 accumulate, M = 128, N = n
__host__ __device__ constexpr uint32_t idesc_bf16(int n, bool a_mn, bool b_mn) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | ((b_mn ? 1u : 0u) << 16) |
           ((uint32_t)(n >> 3) << 17) | ((128u >> 4) << 24);
}

// 16-bit operand panels, SWIZZLE_128B (bf16; input encoder):
//   K-major  (128 rows x 64 K): row r at r*128 B, 16-B chunk c at chunk c ^ (r&7); SBO 1024;
//            one MMA (K = 16 = 32 B) starts at base + ks*32.
//   MN-major (128 MN x 64 K): atoms of 64 MN (128 B) x 8 K rows (1024 B), 16-B chunk c of K
//            row kk at chunk c ^ kk; MN atoms 1024 B apart (LBO), 8-row K groups 2048 B apart
//            (SBO); one MMA (K = 16 rows) starts at base + ks*4096.
__device__ __forceinline__ uint32_t kmaj16_chunk(int r, int c) {
    return (uint32_t)(r * 128 + (((c ^ (r & 7)) & 7) << 4));
}
__device__ __forceinline__ uint32_t mnmaj16_chunk(int mn, int k) {   // mn multiple of 8
    const int kk = k & 7, c = (mn & 63) >> 3;
    return (uint32_t)((k >> 3) * 2048 + (mn >> 6) * 1024 + kk * 128 + (((c ^ kk) & 7) << 4));
}
__device__ __forceinline__ uint64_t desc_mnmajor16(uint32_t addr) { return desc_encode(addr, 1024, 2048, 2); }

// byte offset of element (r, k) inside a K-major panel (k in [0,32))
__device__ __forceinline__ uint32_t kmajor_off(int r, int k) {
    return (uint32_t)(r * 128 + ((((k >> 2) ^ (r & 7)) & 7) << 4) + ((k & 3) << 2));
}
// byte offset of element (mn, k) inside an MN-major panel (mn in [0,128), k in [0,32))
__device__ __forceinline__ uint32_t mnmajor_off(int mn, int k) {
    return (uint32_t)((k >> 2) * 2048 + (mn >> 5) * 512 + (k & 3) * 128 +
                      (((((mn & 31) >> 3) ^ (k & 3)) & 3) << 5) + ((mn & 7) << 2));
}

// ---- tf32 split for 3xTF32 -----------------------------------------------------------
__device__ __forceinline__ uint32_t to_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r;
}
// rna tf32 rounding with integer ops (same result as cvt.rna.tf32.f32 for finite x): add half
// an ulp of the kept 10-bit mantissa, then drop the 13 low bits.  Runs on the ALU pipes
// instead of the narrower conversion pipe.
__device__ __forceinline__ uint32_t rna_tf32_bits(uint32_t b) { return (b + 0x1000u) & 0xFFFFE000u; }
__device__ __forceinline__ void split_tf32(float x, uint32_t& hi, uint32_t& lo) {
    hi = rna_tf32_bits(__float_as_uint(x));
    lo = rna_tf32_bits(__float_as_uint(x - __uint_as_float(hi)));
}

// ---- cp.async (LDGSTS) with zero fill ------------------------------------------------
__device__ __forceinline__ void cp16(uint32_t dst, const void* src, int bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp4(uint32_t dst, const void* src, int bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// ---- mbarrier ------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t a = smem_u32(bar);
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(a),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// ---- TMEM ------------------------------------------------------------------------------
template <int NCOLS>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem) {   // one full warp
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "n"(NCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
template <int NCOLS>
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr) {     // same warp
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "n"(NCOLS) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// ---- MMA -----------------------------------------------------------------------------
__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(accum)
        : "memory");
}
__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t accum) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(da), "l"(db), "r"(idesc), "r"(accum)
        : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

// 32 lanes x 32 consecutive 32-bit columns: thread i of the warp gets row (lane base + i)
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr)
        : "memory");
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

}  // namespace umma
}  // namespace gsb
