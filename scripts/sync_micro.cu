// sync_micro.cu -- cycle costs of the synchronisation / async primitives the warp-specialized
// GEMM pipelines use (one CTA, clock64; tools, not product code).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 -I paper_2406_06022_b200/csrc
//      scripts/sync_micro.cu -o scripts/sync_micro.bin
#include <cuda_runtime.h>
#include <stdio.h>

#include "umma.cuh"

using namespace gsb;

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(umma::smem_u32(b)) : "memory");
}

constexpr int N = 256;

__global__ void micro(long long* out, unsigned long long* sink) {
    __shared__ __align__(8) uint64_t b0, b1, b2;
    __shared__ __align__(1024) float buf[10240];
    __shared__ uint32_t tm;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        umma::mbar_init(&b0, 1);
        umma::mbar_init(&b1, 1);
        umma::mbar_init(&b2, 1);
        umma::fence_barrier_init();
    }
    if (warp == 0) umma::tmem_alloc<128>(&tm);
    umma::tc_fence_before();
    __syncthreads();
    umma::tc_fence_after();
    unsigned long long acc = 0;
    // 0: globaltimer read
    if (tid == 0) {
        long long c0 = clock64();
        for (int i = 0; i < N; ++i) acc += gtimer();
        out[0] = (clock64() - c0) / N;
        // 1: SM clock vs globaltimer (MHz)
        unsigned long long g0 = gtimer();
        c0 = clock64();
        while (gtimer() - g0 < 20000) {
        }
        out[1] = (clock64() - c0) * 1000 / (long long)(gtimer() - g0);
    }
    __syncthreads();
    // 2: warp 0 <-> warp 1 ping-pong through two mbarriers (round trip)
    if (lane == 0 && warp < 2) {
        long long c0 = clock64();
        for (int i = 0; i < N; ++i) {
            if (warp == 0) {
                arrive(&b0);
                umma::mbar_wait(&b1, i & 1);
            } else {
                umma::mbar_wait(&b0, i & 1);
                arrive(&b1);
            }
        }
        if (warp == 0) out[2] = (clock64() - c0) / N;
    }
    __syncthreads();
    // 3: tcgen05.commit (no MMA in flight) -> wait, one thread
    if (tid == 0) {
        long long c0 = clock64();
        for (int i = 0; i < N; ++i) {
            umma::mma_commit(&b2);
            umma::mbar_wait(&b2, i & 1);
        }
        out[3] = (clock64() - c0) / N;
    }
    __syncthreads();
    // 4: fence.proxy.async.shared::cta after one STS per thread, 128 threads
    if (tid < 128) {
        long long c0 = clock64();
        for (int i = 0; i < N; ++i) {
            buf[tid * 4 + (i & 3)] = (float)i;
            umma::fence_proxy_async_smem();
        }
        if (tid == 0) out[4] = (clock64() - c0) / N;
    }
    __syncthreads();
    // 5: named barrier among 128 threads
    if (tid < 128) {
        long long c0 = clock64();
        for (int i = 0; i < N; ++i) asm volatile("bar.sync 2, 128;" ::: "memory");
        if (tid == 0) out[5] = (clock64() - c0) / N;
    }
    __syncthreads();
    // 6: tcgen05.ld 32x32b.x32 + wait (warps 0-3, own lane quarter)
    if (tid < 128) {
        float v[32];
        long long c0 = clock64();
        for (int i = 0; i < N; ++i) {
            umma::tmem_ld32(tm + ((uint32_t)(warp * 32) << 16) + (i & 3) * 32, v);
            acc += __float_as_uint(v[i & 31]);
        }
        if (tid == 0) out[6] = (clock64() - c0) / N;
    }
    __syncthreads();
    // 7: 8 STS.128 per thread (SW128 rows) + fence + bar: the epilogue staging step
    if (tid < 128) {
        const uint32_t base = umma::smem_u32(buf);
        long long c0 = clock64();
        for (int i = 0; i < N; ++i) {
#pragma unroll
            for (int e = 0; e < 32; e += 4)
                asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(base + umma::kmajor_off(tid, e)),
                             "r"(i)
                             : "memory");
            umma::fence_proxy_async_smem();
            asm volatile("bar.sync 2, 128;" ::: "memory");
        }
        if (tid == 0) out[7] = (clock64() - c0) / N;
    }
    __syncthreads();
    // 8: mbarrier try_wait on an already-completed phase
    if (tid == 0) {
        long long c0 = clock64();
        for (int i = 0; i < N; ++i) umma::mbar_wait(&b2, ((N - 1) & 1));
        out[8] = (clock64() - c0) / N;
    }
    // 9-12: tcgen05.mma throughput (SS operands from smem garbage, one thread issues 96, commit, wait)
    if (tid == 0) {
        const uint32_t a0 = umma::smem_u32(buf), b0 = a0 + 16384;
        const uint64_t da = umma::desc_kmajor(a0), db = umma::desc_kmajor(b0);
        const int NM = 96;
        // 9: tf32 M128 N128 K8, SS
        long long c0 = clock64();
        for (int i = 0; i < NM; ++i) umma::mma_tf32(tm, da, db, umma::idesc_tf32(128, false, false), 1u);
        umma::mma_commit(&b2);
        umma::mbar_wait(&b2, 0);
        out[9] = (clock64() - c0) / NM;
        // 10: bf16 M128 N128 K16, SS
        c0 = clock64();
        for (int i = 0; i < NM; ++i) umma::mma_f16(tm, da, db, umma::idesc_bf16(128, false, false), 1u);
        umma::mma_commit(&b2);
        umma::mbar_wait(&b2, 1);
        out[10] = (clock64() - c0) / NM;
        // 11: tf32 M128 N64 K8, SS
        c0 = clock64();
        for (int i = 0; i < NM; ++i) umma::mma_tf32(tm, da, db, umma::idesc_tf32(64, false, false), 1u);
        umma::mma_commit(&b2);
        umma::mbar_wait(&b2, 0);
        out[11] = (clock64() - c0) / NM;
        // 12: tf32 M128 N128 K8, A from TMEM (columns 0..7 of the allocation)
        c0 = clock64();
        for (int i = 0; i < NM; ++i) {
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm + 64),
                "r"(tm), "l"(db), "r"(umma::idesc_tf32(64, false, false)), "r"(1u)
                : "memory");
        }
        umma::mma_commit(&b2);
        umma::mbar_wait(&b2, 1);
        out[12] = (clock64() - c0) / NM;
    }
    sink[tid] = acc;
    umma::tc_fence_before();
    __syncthreads();
    if (warp == 0) umma::tmem_dealloc<128>(tm);
}

int main() {
    long long* d;
    unsigned long long* s;
    cudaMalloc(&d, 64 * 8);
    cudaMalloc(&s, 1024 * 8);
    for (int rep = 0; rep < 3; ++rep) micro<<<1, 256>>>(d, s);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[16];
    cudaMemcpy(h, d, 13 * 8, cudaMemcpyDeviceToHost);
    printf("err %s\n", cudaGetErrorString(e));
    const char* names[] = {"globaltimer read",        "SM clock MHz (clock64 vs globaltimer)",
                           "mbarrier ping-pong (round trip, 2 warps)", "tcgen05.commit -> wait (no MMA)",
                           "STS + fence.proxy.async (128 thr)",     "bar.sync 2,128",
                           "tcgen05.ld 32x32b.x32 + wait",          "8 STS.128 + fence + bar (epilogue staging)",
                           "try_wait on completed phase",
                           "mma tf32 128x128x8 SS (per instr)", "mma bf16 128x128x16 SS (per instr)",
                           "mma tf32 128x64x8 SS (per instr)", "mma tf32 128x64x8 A-in-TMEM (per instr)"};
    for (int i = 0; i < 13; ++i) printf("%-45s %lld cycles\n", names[i], h[i]);
    return 0;
}
