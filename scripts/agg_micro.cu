// Aggregation design study (mag layer-0 shape): n_dst rows x S slots, segment lengths
// uniform in [0, F], source rows = bf16 128-d (256 B) rows of a 1.94M-row table picked at
// random; output Acat fp32 [n_dst][(S+1)*128] = per-slot means + self row.
// Variants: v0 = warp per row, slot by slot (the shipped kernel's structure);
// v2 = half-warp per row (two rows per warp, independent); v3 = quarter... ; ceiling = the same
// rows gathered in edge order with no segments.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1;}}while(0)

constexpr int D = 128, S = 3;
__device__ __forceinline__ void acc8(float* a, uint4 x) {
    a[0] += __uint_as_float(x.x << 16); a[1] += __uint_as_float(x.x & 0xffff0000u);
    a[2] += __uint_as_float(x.y << 16); a[3] += __uint_as_float(x.y & 0xffff0000u);
    a[4] += __uint_as_float(x.z << 16); a[5] += __uint_as_float(x.z & 0xffff0000u);
    a[6] += __uint_as_float(x.w << 16); a[7] += __uint_as_float(x.w & 0xffff0000u);
}

// v0: warp per row; per slot: keys (<=32) by one load; LPE=16 lanes per row, 2 edges per pass, U per lane
template <int U>
__global__ void __launch_bounds__(256) v0(const uint4* __restrict__ tab, const int64_t* __restrict__ seg,
                                          const int64_t* __restrict__ key, const int64_t* __restrict__ self,
                                          int n, float* __restrict__ out) {
    const int lane = threadIdx.x & 31, grp = lane >> 4, sub = lane & 15;
    const int warps = gridDim.x * blockDim.x >> 5;
    for (int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < n; j += warps) {
        const int64_t bl = lane <= S ? seg[(int64_t)j * S + lane] : 0;
        const uint4 xs = __ldg(tab + self[j] * 16 + sub);
        float* o = out + (int64_t)j * (S + 1) * D;
        for (int s = 0; s < S; ++s) {
            const int64_t e0 = __shfl_sync(~0u, bl, s), e1 = __shfl_sync(~0u, bl, s + 1);
            float a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            for (int64_t cb = e0; cb < e1; cb += 32) {
                const int64_t k = cb + lane < e1 ? key[cb + lane] : 0;
                const int cnt = (int)min((int64_t)32, e1 - cb);
                for (int kk = 0; kk < cnt; kk += 2 * U) {
                    uint4 x[U];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        const int idx = kk + grp + 2 * u;
                        const int64_t r = __shfl_sync(~0u, k, idx & 31);
                        x[u] = idx < cnt ? __ldg(tab + r * 16 + sub) : make_uint4(0, 0, 0, 0);
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) acc8(a, x[u]);
                }
            }
#pragma unroll
            for (int v = 0; v < 8; ++v) a[v] += __shfl_xor_sync(~0u, a[v], 16);
            const float inv = e1 > e0 ? 1.f / (float)(e1 - e0) : 0.f;
            if (grp == 0) {
                float4* p = reinterpret_cast<float4*>(o + s * D + sub * 8);
                p[0] = make_float4(a[0] * inv, a[1] * inv, a[2] * inv, a[3] * inv);
                p[1] = make_float4(a[4] * inv, a[5] * inv, a[6] * inv, a[7] * inv);
            }
        }
        if (grp == 0) {
            float a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            acc8(a, xs);
            float4* p = reinterpret_cast<float4*>(o + S * D + sub * 8);
            p[0] = make_float4(a[0], a[1], a[2], a[3]);
            p[1] = make_float4(a[4], a[5], a[6], a[7]);
        }
    }
}

// v2: half-warp per row (rows j, j+1 in the two halves), all slots' edges of the row loaded
// up front (<= 16 keys per half-warp pass), U rows in flight per lane, per-slot running sums
// closed at slot boundaries (half-warp-uniform), no cross-half reduction.
template <int U>
__global__ void __launch_bounds__(256) v2(const uint4* __restrict__ tab, const int64_t* __restrict__ seg,
                                          const int64_t* __restrict__ key, const int64_t* __restrict__ self,
                                          int n, float* __restrict__ out) {
    const int lane = threadIdx.x & 31, half = lane >> 4, sub = lane & 15;
    const unsigned hm = half ? 0xffff0000u : 0x0000ffffu;
    const int hw = (gridDim.x * blockDim.x) >> 4;
    for (int j = (blockIdx.x * blockDim.x + threadIdx.x) >> 4; j < n; j += hw) {
        const int64_t bl = sub <= S ? seg[(int64_t)j * S + sub] : 0;
        const uint4 xs = __ldg(tab + self[j] * 16 + sub);
        float* o = out + (int64_t)j * (S + 1) * D;
        const int64_t eb = __shfl_sync(hm, bl, 0, 16), ee = __shfl_sync(hm, bl, S, 16);
        int s = 0;
        int64_t sb = eb, se = __shfl_sync(hm, bl, 1, 16);
        float a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int64_t cb = eb; cb < ee; cb += 16) {
            const int64_t k = cb + sub < ee ? key[cb + sub] : 0;
            const int cnt = (int)min((int64_t)16, ee - cb);
            for (int kk = 0; kk < cnt; kk += U) {
                uint4 x[U];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int64_t r = __shfl_sync(hm, k, (kk + u) & 15, 16);
                    x[u] = kk + u < cnt ? __ldg(tab + r * 16 + sub) : make_uint4(0, 0, 0, 0);
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (kk + u < cnt) {
                        const int64_t e = cb + kk + u;
                        while (e >= se) {
                            const float inv = se > sb ? 1.f / (float)(se - sb) : 0.f;
                            float4* p = reinterpret_cast<float4*>(o + s * D + sub * 8);
                            p[0] = make_float4(a[0] * inv, a[1] * inv, a[2] * inv, a[3] * inv);
                            p[1] = make_float4(a[4] * inv, a[5] * inv, a[6] * inv, a[7] * inv);
#pragma unroll
                            for (int v = 0; v < 8; ++v) a[v] = 0.f;
                            ++s;
                            sb = se;
                            se = __shfl_sync(hm, bl, s + 1, 16);
                        }
                        acc8(a, x[u]);
                    }
                }
            }
        }
        for (; s < S; ++s) {
            const float inv = se > sb ? 1.f / (float)(se - sb) : 0.f;
            float4* p = reinterpret_cast<float4*>(o + s * D + sub * 8);
            p[0] = make_float4(a[0] * inv, a[1] * inv, a[2] * inv, a[3] * inv);
            p[1] = make_float4(a[4] * inv, a[5] * inv, a[6] * inv, a[7] * inv);
#pragma unroll
            for (int v = 0; v < 8; ++v) a[v] = 0.f;
            sb = se;
            se = __shfl_sync(hm, bl, min(s + 2, S), 16);
        }
        float b[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        acc8(b, xs);
        float4* p = reinterpret_cast<float4*>(o + S * D + sub * 8);
        p[0] = make_float4(b[0], b[1], b[2], b[3]);
        p[1] = make_float4(b[4], b[5], b[6], b[7]);
    }
}

// ceiling: the same E rows in edge order, 16 lanes per row, U per lane, sum only
template <int U>
__global__ void __launch_bounds__(256) ceil_k(const uint4* __restrict__ tab, const int64_t* __restrict__ key, int64_t E,
                                              float* __restrict__ out) {
    const int lane = threadIdx.x & 31, grp = lane >> 4, sub = lane & 15;
    const int64_t warps = (gridDim.x * (int64_t)blockDim.x) >> 5;
    float a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t b = ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) * (2 * U); b < E; b += warps * 2 * U) {
        const int64_t k = (lane < 2 * U && b + lane < E) ? key[b + lane] : 0;
        uint4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t r = __shfl_sync(~0u, k, grp + 2 * u);
            x[u] = b + grp + 2 * u < E ? __ldg(tab + r * 16 + sub) : make_uint4(0, 0, 0, 0);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc8(a, x[u]);
    }
    if (a[0] == 1.2345f) out[0] = a[1];
}

int main() {
    const int64_t NT = 1939743;             // table rows (mag nodes), 256 B each
    const int n = 16800, F = 15;
    std::mt19937_64 rng(1);
    std::vector<int64_t> seg((size_t)n * S + 1), self(n), key;
    seg[0] = 0;
    for (int64_t q = 0; q < (int64_t)n * S; ++q) {
        const int len = (q % S == 2 && (q / S) % 3 == 0) ? 0 : (int)(rng() % (F + 1));
        seg[q + 1] = seg[q] + len;
    }
    const int64_t E = seg.back();
    key.resize(E);
    for (auto& k : key) k = (int64_t)(rng() % NT);
    for (auto& s : self) s = (int64_t)(rng() % NT);
    printf("n_dst %d, edges %lld (%.1f per row)\n", n, (long long)E, (double)E / n);
    uint4* tab; int64_t *dseg, *dkey, *dself; float* out; char* flush;
    CK(cudaMalloc(&tab, NT * 256)); CK(cudaMemset(tab, 0x3f, NT * 256));
    CK(cudaMalloc(&dseg, seg.size() * 8)); CK(cudaMalloc(&dkey, E * 8)); CK(cudaMalloc(&dself, n * 8));
    CK(cudaMalloc(&out, (size_t)n * (S + 1) * D * 4)); CK(cudaMalloc(&flush, 256 << 20));
    CK(cudaMemcpy(dseg, seg.data(), seg.size() * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dkey, key.data(), E * 8, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dself, self.data(), n * 8, cudaMemcpyHostToDevice));
    const double alg = (double)E * (256 + 8) + (double)n * (256 + (S + 1) * D * 4 + (S + 1) * 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&](const char* name, auto launch) {
        float best = 1e9;
        for (int it = 0; it < 8; ++it) {
            cudaMemsetAsync(flush, it, 256 << 20);
            cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); if (it > 1 && ms < best) best = ms;
        }
        printf("%-28s %7.1f us  %6.0f GB/s alg  %s\n", name, best * 1e3, alg / (best * 1e-3) / 1e9,
               cudaGetErrorString(cudaGetLastError()));
    };
    char nm[64];
    for (int mb : {4, 6, 8}) {
        snprintf(nm, 64, "v0 U4 blocks/SM %d", mb); run(nm, [&] { v0<4><<<148 * mb, 256>>>(tab, dseg, dkey, dself, n, out); });
        snprintf(nm, 64, "v0 U8 blocks/SM %d", mb); run(nm, [&] { v0<8><<<148 * mb, 256>>>(tab, dseg, dkey, dself, n, out); });
        snprintf(nm, 64, "v2 U4 blocks/SM %d", mb); run(nm, [&] { v2<4><<<148 * mb, 256>>>(tab, dseg, dkey, dself, n, out); });
        snprintf(nm, 64, "v2 U8 blocks/SM %d", mb); run(nm, [&] { v2<8><<<148 * mb, 256>>>(tab, dseg, dkey, dself, n, out); });
    }
    int g2 = (n * 16 + 255) / 256;
    snprintf(nm, 64, "v2 U4 one row per half-warp"); run(nm, [&] { v2<4><<<g2, 256>>>(tab, dseg, dkey, dself, n, out); });
    snprintf(nm, 64, "v2 U8 one row per half-warp"); run(nm, [&] { v2<8><<<g2, 256>>>(tab, dseg, dkey, dself, n, out); });
    int g0 = (n * 32 + 255) / 256;
    snprintf(nm, 64, "v0 U4 one row per warp"); run(nm, [&] { v0<4><<<g0, 256>>>(tab, dseg, dkey, dself, n, out); });
    for (int mb : {4, 8}) {
        snprintf(nm, 64, "ceiling U4 blocks/SM %d", mb); run(nm, [&] { ceil_k<4><<<148 * mb, 256>>>(tab, dkey, E, out); });
    }
    const double gath = (double)E * 264;
    printf("(ceiling GB/s above counts segment-free bytes %.1f MB as alg %.1f MB)\n", gath / 1e6, alg / 1e6);
    return 0;
}
