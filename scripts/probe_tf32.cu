// probe_tf32.cu -- one-CTA probes for the next TMA GEMM design (tools, not product code).
//   (a) does kind::tf32 read a raw fp32 operand as its truncation to tf32 (low 13 mantissa bits
//       ignored)?  D(raw, raw) is compared bit-for-bit with D(trunc, trunc) and D(rna, rna).
//   (b) the smem image of a TMA load with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, box {32, 32} of a
//       plain [32 k][128 mn] fp32 matrix: where element (k, mn) lands (dumped, decoded on host).
//   (c) TMA reduce-add (cp.reduce.async.bulk.tensor .add, f32) of a SWIZZLE_128B [128][32] tile.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2406_06022_b200/csrc
//      scripts/probe_tf32.cu -o /tmp/probe_tf32 -lcuda
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <vector>

#include "umma.cuh"

using namespace gsb;

#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e = (x);                                                           \
        if (e != cudaSuccess) {                                                        \
            fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
            exit(1);                                                                   \
        }                                                                              \
    } while (0)

__device__ uint32_t trunc_bits(float x) { return __float_as_uint(x) & 0xFFFFE000u; }

// (a): mode 0 raw, 1 trunc, 2 rna.  A, B: [128][32] fp32 row-major (K contiguous).  D [128][128].
__global__ void probe_a(const float* A, const float* B, int mode, float* D) {
    __shared__ __align__(1024) uint8_t sm[2 * 16384];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tm;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 128 * 32; i += blockDim.x) {
        const int r = i / 32, k = i % 32;
        float a = A[i], b = B[i];
        uint32_t ua = __float_as_uint(a), ub = __float_as_uint(b);
        if (mode == 1) { ua = trunc_bits(a); ub = trunc_bits(b); }
        if (mode == 2) { ua = umma::rna_tf32_bits(ua); ub = umma::rna_tf32_bits(ub); }
        *reinterpret_cast<uint32_t*>(sm + umma::kmajor_off(r, k)) = ua;
        *reinterpret_cast<uint32_t*>(sm + 16384 + umma::kmajor_off(r, k)) = ub;
    }
    if (tid == 0) { umma::mbar_init(&bar, 1); umma::fence_barrier_init(); }
    if (warp == 0) umma::tmem_alloc<128>(&tm);
    umma::fence_proxy_async_smem();
    umma::tc_fence_before();
    __syncthreads();
    umma::tc_fence_after();
    const uint32_t t = tm;
    if (tid == 0) {
        const uint32_t a0 = umma::smem_u32(sm), b0 = a0 + 16384;
        for (int ks = 0; ks < 4; ++ks)
            umma::mma_tf32(t, umma::desc_kmajor(a0 + ks * 32), umma::desc_kmajor(b0 + ks * 32),
                           umma::idesc_tf32(128, false, false), ks > 0);
        umma::mma_commit(&bar);
    }
    umma::mbar_wait(&bar, 0);
    umma::tc_fence_after();
    for (int c = 0; c < 4; ++c) {
        float v[32];
        umma::tmem_ld32(t + ((uint32_t)(warp * 32) << 16) + c * 32, v);
        for (int j = 0; j < 32; ++j) D[(warp * 32 + (tid & 31)) * 128 + c * 32 + j] = v[j];
    }
    umma::tc_fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc<128>(t);
}

// (b) / (c)
__global__ void probe_b(const __grid_constant__ CUtensorMap m, float* out) {
    __shared__ __align__(1024) uint8_t sm[4096];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        umma::mbar_init(&bar, 1);
        umma::fence_barrier_init();
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(umma::smem_u32(&bar)), "r"(4096)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                umma::smem_u32(sm)),
            "l"(reinterpret_cast<uint64_t>(&m)), "r"(0), "r"(0), "r"(umma::smem_u32(&bar))
            : "memory");
    }
    __syncthreads();
    umma::mbar_wait(&bar, 0);
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) out[i] = reinterpret_cast<float*>(sm)[i];
}

__global__ void probe_c(const __grid_constant__ CUtensorMap m, int n_rep) {
    __shared__ __align__(1024) float sm[128 * 32];
    for (int i = threadIdx.x; i < 128 * 32; i += blockDim.x) {
        const int r = i / 32, k = i % 32;
        *reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(sm) + umma::kmajor_off(r, k)) = (float)(r * 32 + k);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 0; q < n_rep; ++q)
            asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                             reinterpret_cast<uint64_t>(&m)),
                         "r"(0), "r"(0), "r"(umma::smem_u32(sm))
                         : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

// (d) MN-major operands straight from TMA (SWIZZLE_128B_ATOM_32B, box {32 mn, 32 k} per 32-MN
// atom at atom*4096): D = A B with A K-major (or MN-major if a_mn) and B MN-major.  desc LBO/SBO
// given.  At: [32 k][128 m] if a_mn else [128 m][32 k]; Bt: [32 k][128 n].
__global__ void probe_d(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB, const float* A,
                        int a_mn, uint32_t lbo, uint32_t sbo, float* D) {
    __shared__ __align__(1024) uint8_t sm[2 * 16384];
    __shared__ __align__(8) uint64_t bar, bar2;
    __shared__ uint32_t tm;
    const int tid = threadIdx.x, warp = tid >> 5;
    if (!a_mn)
        for (int i = tid; i < 128 * 32; i += blockDim.x)
            *reinterpret_cast<float*>(sm + umma::kmajor_off(i / 32, i % 32)) = A[i];
    if (tid == 0) {
        umma::mbar_init(&bar, 1);
        umma::mbar_init(&bar2, 1);
        umma::fence_barrier_init();
        const uint32_t nb = a_mn ? 32768 : 16384;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(umma::smem_u32(&bar)), "r"(nb)
                     : "memory");
        for (int j = 0; j < 4; ++j) {
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                    umma::smem_u32(sm + 16384 + j * 4096)),
                "l"(reinterpret_cast<uint64_t>(&mB)), "r"(j * 32), "r"(0), "r"(umma::smem_u32(&bar))
                : "memory");
            if (a_mn)
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                        umma::smem_u32(sm + j * 4096)),
                    "l"(reinterpret_cast<uint64_t>(&mA)), "r"(j * 32), "r"(0), "r"(umma::smem_u32(&bar))
                    : "memory");
        }
    }
    if (warp == 0) umma::tmem_alloc<128>(&tm);
    umma::fence_proxy_async_smem();
    umma::tc_fence_before();
    __syncthreads();
    umma::tc_fence_after();
    umma::mbar_wait(&bar, 0);
    const uint32_t t = tm;
    if (tid == 0) {
        const uint32_t a0 = umma::smem_u32(sm), b0 = a0 + 16384;
        for (int ks = 0; ks < 4; ++ks) {
            const uint64_t da = a_mn ? umma::desc_encode(a0 + ks * 1024, lbo, sbo, 1) : umma::desc_kmajor(a0 + ks * 32);
            const uint64_t db = umma::desc_encode(b0 + ks * 1024, lbo, sbo, 1);
            umma::mma_tf32(t, da, db, umma::idesc_tf32(128, a_mn != 0, true), ks > 0);
        }
        umma::mma_commit(&bar2);
    }
    umma::mbar_wait(&bar2, 0);
    umma::tc_fence_after();
    for (int c = 0; c < 4; ++c) {
        float v[32];
        umma::tmem_ld32(t + ((uint32_t)(warp * 32) << 16) + c * 32, v);
        for (int j = 0; j < 32; ++j) D[(warp * 32 + (tid & 31)) * 128 + c * 32 + j] = v[j];
    }
    umma::tc_fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc<128>(t);
}

// (e) bf16 MN-major B straight from TMA SWIZZLE_128B boxes {64 mn, 64 k} (2 boxes 8192 B apart):
// D[128 m][128 n] = A[m][k] B[k][n], K = 64; A K-major bf16 (kmaj16 via STS); desc LBO / SBO given.
__global__ void probe_e(const __grid_constant__ CUtensorMap mB, const __nv_bfloat16* A, uint32_t lbo, uint32_t sbo,
                        float* D) {
    __shared__ __align__(1024) uint8_t sm[2 * 16384];
    __shared__ __align__(8) uint64_t bar, bar2;
    __shared__ uint32_t tm;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 128 * 8; i += blockDim.x) {   // 16-B chunks: row r, chunk c (8 bf16)
        const int r = i / 8, c = i % 8;
        *reinterpret_cast<uint4*>(sm + umma::kmaj16_chunk(r, c)) = *reinterpret_cast<const uint4*>(A + r * 64 + c * 8);
    }
    if (tid == 0) {
        umma::mbar_init(&bar, 1);
        umma::mbar_init(&bar2, 1);
        umma::fence_barrier_init();
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(umma::smem_u32(&bar)), "r"(16384)
                     : "memory");
        for (int j = 0; j < 2; ++j)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                    umma::smem_u32(sm + 16384 + j * 8192)),
                "l"(reinterpret_cast<uint64_t>(&mB)), "r"(j * 64), "r"(0), "r"(umma::smem_u32(&bar))
                : "memory");
    }
    if (warp == 0) umma::tmem_alloc<128>(&tm);
    umma::fence_proxy_async_smem();
    umma::tc_fence_before();
    __syncthreads();
    umma::tc_fence_after();
    umma::mbar_wait(&bar, 0);
    const uint32_t t = tm;
    if (tid == 0) {
        const uint32_t a0 = umma::smem_u32(sm), b0 = a0 + 16384;
        for (int ks = 0; ks < 4; ++ks)
            umma::mma_f16(t, umma::desc_kmajor(a0 + ks * 32), umma::desc_encode(b0 + ks * 2048, lbo, sbo, 2),
                          umma::idesc_bf16(128, false, true), ks > 0);
        umma::mma_commit(&bar2);
    }
    umma::mbar_wait(&bar2, 0);
    umma::tc_fence_after();
    for (int c = 0; c < 4; ++c) {
        float v[32];
        umma::tmem_ld32(t + ((uint32_t)(warp * 32) << 16) + c * 32, v);
        for (int j = 0; j < 32; ++j) D[(warp * 32 + (tid & 31)) * 128 + c * 32 + j] = v[j];
    }
    umma::tc_fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc<128>(t);
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    EncFn enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q));
    // ---- (a)
    std::vector<float> hA(128 * 32), hB(128 * 32);
    srand(7);
    for (auto& x : hA) x = (float)rand() / RAND_MAX * 2.f - 1.f;
    for (auto& x : hB) x = (float)rand() / RAND_MAX * 2.f - 1.f;
    float *dA, *dB, *dD;
    CK(cudaMalloc(&dA, 4 * 4096));
    CK(cudaMalloc(&dB, 4 * 4096));
    CK(cudaMalloc(&dD, 3 * 4 * 16384));
    CK(cudaMemcpy(dA, hA.data(), 4 * 4096, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, hB.data(), 4 * 4096, cudaMemcpyHostToDevice));
    for (int mode = 0; mode < 3; ++mode) probe_a<<<1, 128>>>(dA, dB, mode, dD + mode * 16384);
    CK(cudaDeviceSynchronize());
    std::vector<float> D(3 * 16384);
    CK(cudaMemcpy(D.data(), dD, 4 * 3 * 16384, cudaMemcpyDeviceToHost));
    int eq_tr = 0, eq_rn = 0;
    double maxd = 0, maxerr_raw = 0;
    for (int i = 0; i < 16384; ++i) {
        eq_tr += (memcmp(&D[i], &D[16384 + i], 4) == 0);
        eq_rn += (memcmp(&D[i], &D[2 * 16384 + i], 4) == 0);
        const int r = i / 128, c = i % 128;
        double ref = 0;
        for (int k = 0; k < 32; ++k) ref += (double)hA[r * 32 + k] * hB[c * 32 + k];
        maxerr_raw = fmax(maxerr_raw, fabs(D[i] - ref));
        maxd = fmax(maxd, fabs(ref));
    }
    printf("(a) raw==trunc %d/16384  raw==rna %d/16384  max|raw-exact| %.3g (max|exact| %.3g)\n", eq_tr, eq_rn,
           maxerr_raw, maxd);
    // ---- (b)
    std::vector<float> hM(32 * 128);
    for (int k = 0; k < 32; ++k)
        for (int mn = 0; mn < 128; ++mn) hM[k * 128 + mn] = (float)(k * 1000 + mn);
    float *dM, *dO;
    CK(cudaMalloc(&dM, 4 * 4096));
    CK(cudaMalloc(&dO, 4 * 1024));
    CK(cudaMemcpy(dM, hM.data(), 4 * 4096, cudaMemcpyHostToDevice));
    for (int sw = 3; sw <= 5; ++sw) {
        CUtensorMap m;
        const cuuint64_t dims[2] = {128, 32};
        const cuuint64_t str[1] = {128 * 4};
        const cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
        CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dM, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         (CUtensorMapSwizzle)sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) {
            printf("(b) swizzle %d: encode failed %d\n", sw, (int)r);
            continue;
        }
        probe_b<<<1, 128>>>(m, dO);
        CK(cudaDeviceSynchronize());
        std::vector<float> o(1024);
        CK(cudaMemcpy(o.data(), dO, 4096, cudaMemcpyDeviceToHost));
        printf("(b) swizzle %d: smem float index -> (k, mn)\n", sw);
        for (int row = 0; row < 32; ++row) {   // 128-B rows of smem
            printf("  row %2d:", row);
            for (int c = 0; c < 32; c += 4) {
                const int v = (int)o[row * 32 + c];
                printf(" (%d,%d)", v / 1000, v % 1000);
            }
            printf("\n");
        }
    }
    // ---- (c)
    {
        float* dC;
        CK(cudaMalloc(&dC, 4 * 128 * 40));
        CK(cudaMemset(dC, 0, 4 * 128 * 40));
        CUtensorMap m;
        const cuuint64_t dims[2] = {32, 128};
        const cuuint64_t str[1] = {40 * 4};
        const cuuint32_t box[2] = {32, 128}, es[2] = {1, 1};
        CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dC, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("(c) encode %d\n", (int)r);
        probe_c<<<1, 128>>>(m, 3);
        CK(cudaDeviceSynchronize());
        std::vector<float> c(128 * 40);
        CK(cudaMemcpy(c.data(), dC, 4 * 128 * 40, cudaMemcpyDeviceToHost));
        int ok = 0;
        for (int rr = 0; rr < 128; ++rr)
            for (int k = 0; k < 40; ++k) ok += (c[rr * 40 + k] == (k < 32 ? 3.f * (rr * 32 + k) : 0.f));
        printf("(c) reduce-add x3 correct %d/%d\n", ok, 128 * 40);
    }
    // ---- (d)
    {
        // A [128 m][32 k], At [32 k][128 m], Bt [32 k][128 n]
        std::vector<float> At(32 * 128), Bt(32 * 128);
        for (int m = 0; m < 128; ++m)
            for (int k = 0; k < 32; ++k) At[k * 128 + m] = hA[m * 32 + k];
        for (int n = 0; n < 128; ++n)
            for (int k = 0; k < 32; ++k) Bt[k * 128 + n] = hB[n * 32 + k];
        float *dAt, *dBt;
        CK(cudaMalloc(&dAt, 4 * 4096));
        CK(cudaMalloc(&dBt, 4 * 4096));
        CK(cudaMemcpy(dAt, At.data(), 4 * 4096, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dBt, Bt.data(), 4 * 4096, cudaMemcpyHostToDevice));
        CUtensorMap ma, mb;
        const cuuint64_t dims[2] = {128, 32};
        const cuuint64_t str[1] = {128 * 4};
        const cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
        CUresult r1 = enc(&ma, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dAt, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        CUresult r2 = enc(&mb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dBt, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("(d) encode %d %d\n", (int)r1, (int)r2);
        const uint32_t lbos[2] = {4096, 512}, sbos[2] = {512, 4096};
        for (int a_mn = 0; a_mn < 2; ++a_mn)
            for (int v = 0; v < 2; ++v) {
                probe_d<<<1, 128>>>(ma, mb, dA, a_mn, lbos[v], sbos[v], dD);
                CK(cudaDeviceSynchronize());
                CK(cudaMemcpy(D.data(), dD, 4 * 16384, cudaMemcpyDeviceToHost));
                double me = 0;
                for (int i = 0; i < 16384; ++i) {
                    const int rr = i / 128, c = i % 128;
                    double ref = 0;
                    for (int k = 0; k < 32; ++k) ref += (double)hA[rr * 32 + k] * hB[c * 32 + k];
                    me = fmax(me, fabs(D[i] - ref));
                }
                printf("(d) a_mn %d lbo %u sbo %u: max|D-exact| %.3g\n", a_mn, lbos[v], sbos[v], me);
            }
    }
    // ---- (e)
    {
        std::vector<__nv_bfloat16> Ab(128 * 64), Bt(64 * 128);   // A [m][k], Bt [k][n]
        std::vector<float> Af(128 * 64), Bf(64 * 128);
        for (int i = 0; i < 128 * 64; ++i) { Ab[i] = __float2bfloat16((float)rand() / RAND_MAX - 0.5f); Af[i] = __bfloat162float(Ab[i]); }
        for (int i = 0; i < 64 * 128; ++i) { Bt[i] = __float2bfloat16((float)rand() / RAND_MAX - 0.5f); Bf[i] = __bfloat162float(Bt[i]); }
        __nv_bfloat16 *dAb, *dBt;
        CK(cudaMalloc(&dAb, 2 * 8192));
        CK(cudaMalloc(&dBt, 2 * 8192));
        CK(cudaMemcpy(dAb, Ab.data(), 2 * 8192, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dBt, Bt.data(), 2 * 8192, cudaMemcpyHostToDevice));
        CUtensorMap mb;
        const cuuint64_t dims[2] = {128, 64};
        const cuuint64_t str[1] = {128 * 2};
        const cuuint32_t box[2] = {64, 64}, es[2] = {1, 1};
        CUresult r = enc(&mb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dBt, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("(e) encode %d\n", (int)r);
        const uint32_t lbos[2] = {8192, 1024}, sbos[2] = {1024, 8192};
        for (int v = 0; v < 2; ++v) {
            probe_e<<<1, 128>>>(mb, dAb, lbos[v], sbos[v], dD);
            CK(cudaDeviceSynchronize());
            CK(cudaMemcpy(D.data(), dD, 4 * 16384, cudaMemcpyDeviceToHost));
            double me = 0;
            for (int i = 0; i < 16384; ++i) {
                const int rr = i / 128, c = i % 128;
                double ref = 0;
                for (int k = 0; k < 64; ++k) ref += (double)Af[rr * 64 + k] * Bf[k * 128 + c];
                me = fmax(me, fabs(D[i] - ref));
            }
            printf("(e) bf16 MN-major B lbo %u sbo %u: max|D-exact| %.3g\n", lbos[v], sbos[v], me);
        }
    }
    return 0;
}
