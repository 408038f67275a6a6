// probe_bf16.cu -- checks the tcgen05 kind::f16 (bf16) operand layouts used by the input
// encoder: K-major SWIZZLE_128B for A and B (forward) and MN-major SWIZZLE_128B for A and B
// (weight-gradient), on one 128 x 128 x 64 block against a CPU reference.
// Build + run (GPU box): nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 \
//   -I paper_2406_06022_b200/csrc -I include scripts/probe_bf16.cu -o /tmp/probe_bf16 && /tmp/probe_bf16
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "umma.cuh"

using namespace gsb;

__device__ uint32_t kmaj_off16(int r, int k) {   // 128 rows x 64 bf16, 128-B rows
    return (uint32_t)(r * 128 + ((((k >> 3) ^ (r & 7)) & 7) << 4) + ((k & 7) << 1));
}
__device__ uint32_t mnmaj_off16(int mn, int k, uint32_t lbo, uint32_t sbo) {   // 128 MN x 64 K
    const int atom = mn >> 6, kg = k >> 3, kk = k & 7, c = (mn & 63) >> 3;
    return (uint32_t)(kg * sbo + atom * lbo + kk * 128 + (((c ^ kk) & 7) << 4) + ((mn & 7) << 1));
}

// A: [128][64] row-major (m, k); B: [64][128] row-major (k, n); D = A B  (128 x 128 fp32)
__global__ void probe(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D, int a_mn, int b_mn, uint32_t lbo,
                      uint32_t sbo, int swap) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sa = sm;
    uint8_t* sb = sm + 16384;
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tm;
    const int tid = threadIdx.x;
    for (int i = tid; i < 128 * 64; i += blockDim.x) {
        const int m = i / 64, k = i % 64;
        const uint32_t o = a_mn ? mnmaj_off16(m, k, lbo, sbo) : kmaj_off16(m, k);
        *reinterpret_cast<__nv_bfloat16*>(sa + o) = A[m * 64 + k];
    }
    for (int i = tid; i < 64 * 128; i += blockDim.x) {
        const int k = i / 128, n = i % 128;
        const uint32_t o = b_mn ? mnmaj_off16(n, k, lbo, sbo) : kmaj_off16(n, k);
        *reinterpret_cast<__nv_bfloat16*>(sb + o) = B[k * 128 + n];
    }
    if ((tid >> 5) == 0) umma::tmem_alloc<128>(&tm);
    if (tid == 0) {
        umma::mbar_init(&bar, 1);
        umma::fence_barrier_init();
    }
    umma::fence_proxy_async_smem();
    umma::tc_fence_before();
    __syncthreads();
    umma::tc_fence_after();
    const uint32_t tmem = tm;
    if (tid == 0) {
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
                               ((128u >> 3) << 17) | ((128u >> 4) << 24);
        const uint32_t l = swap ? sbo : lbo, s = swap ? lbo : sbo;
        for (int ks = 0; ks < 4; ++ks) {
            const uint32_t a = umma::smem_u32(sa) + (a_mn ? ks * 2 * sbo : ks * 32);
            const uint32_t b = umma::smem_u32(sb) + (b_mn ? ks * 2 * sbo : ks * 32);
            const uint64_t da = a_mn ? umma::desc_encode(a, l, s, 2) : umma::desc_kmajor(a);
            const uint64_t db = b_mn ? umma::desc_encode(b, l, s, 2) : umma::desc_kmajor(b);
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                "l"(da), "l"(db), "r"(idesc), "r"(ks > 0 ? 1u : 0u)
                : "memory");
        }
        umma::mma_commit(&bar);
    }
    umma::mbar_wait(&bar, 0);
    umma::tc_fence_after();
    const int warp = tid >> 5, lane = tid & 31;
    if (warp < 4) {
        for (int c = 0; c < 4; ++c) {
            float v[32];
            umma::tmem_ld32(tmem + ((uint32_t)(warp * 32) << 16) + c * 32, v);
            for (int j = 0; j < 32; ++j) D[(warp * 32 + lane) * 128 + c * 32 + j] = v[j];
        }
    }
    umma::tc_fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc<128>(tmem);
}

int main() {
    std::vector<__nv_bfloat16> A(128 * 64), B(64 * 128);
    std::vector<float> Af(128 * 64), Bf(64 * 128);
    srand(1);
    for (int i = 0; i < 128 * 64; ++i) {
        float x = (float)(rand() % 255 - 127) / 64.f;
        A[i] = __float2bfloat16(x);
        Af[i] = __bfloat162float(A[i]);
    }
    for (int i = 0; i < 64 * 128; ++i) {
        float x = (float)(rand() % 255 - 127) / 64.f;
        B[i] = __float2bfloat16(x);
        Bf[i] = __bfloat162float(B[i]);
    }
    std::vector<double> ref(128 * 128, 0.0);
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 128; ++n) {
            double s = 0;
            for (int k = 0; k < 64; ++k) s += (double)Af[m * 64 + k] * Bf[k * 128 + n];
            ref[m * 128 + n] = s;
        }
    __nv_bfloat16 *dA, *dB;
    float* dD;
    cudaMalloc(&dA, A.size() * 2);
    cudaMalloc(&dB, B.size() * 2);
    cudaMalloc(&dD, 128 * 128 * 4);
    cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    struct V { int amn, bmn; uint32_t lbo, sbo; int swap; } vs[] = {
        {0, 0, 16, 1024, 0}, {1, 1, 1024, 2048, 0}, {1, 1, 1024, 2048, 1}, {1, 0, 1024, 2048, 0},
        {0, 1, 1024, 2048, 0}};
    std::vector<float> D(128 * 128);
    for (auto& v : vs) {
        cudaMemset(dD, 0, 128 * 128 * 4);
        probe<<<1, 128, 40000>>>(dA, dB, dD, v.amn, v.bmn, v.lbo, v.sbo, v.swap);
        cudaError_t e = cudaDeviceSynchronize();
        cudaMemcpy(D.data(), dD, 128 * 128 * 4, cudaMemcpyDeviceToHost);
        double err = 0;
        for (int i = 0; i < 128 * 128; ++i) err = fmax(err, fabs(D[i] - ref[i]));
        printf("a_mn %d b_mn %d lbo %u sbo %u swap %d: %s max err %.3e (D[0]=%f ref %f)\n", v.amn, v.bmn, v.lbo, v.sbo,
               v.swap, cudaGetErrorString(e), err, D[0], ref[0]);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
