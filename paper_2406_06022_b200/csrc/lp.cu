// lp.cu -- link prediction: joint negative sampling, the LP seed set, DistMult
// scoring (Eq. 3) with contrastive (Eq. 7) or cross-entropy (Eq. 4) loss and gradients.
// Contract: include/gsb.h "Link prediction".
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_select.cuh>

#include "gsb_internal.cuh"
#include "rng.cuh"

namespace gsb {

// Draw i = (key k = key_base + i / K, j = i % K): joint negatives key by group (tag 0xFFF),
// uniform negatives by positive (tag 0xFFE); R-rng.
__global__ void joint_neg_kernel(int64_t total, int K, int64_t n_nodes, int64_t base, uint64_t seed, uint32_t step_host,
                                 const uint32_t* __restrict__ step_dev, int64_t group_base, int64_t* __restrict__ neg,
                                 uint32_t tag) {
    GSB_PDL_ENTRY();
    const uint32_t step = step_dev ? *step_dev : step_host;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = group_base + i / K;
        const uint32_t j = (uint32_t)(i % K);
        uint64_t x = keyed_u64(seed, (uint32_t)(uint64_t)g, (uint32_t)((uint64_t)g >> 32), tag | (j & 0xFFFFu), step);
        neg[i] = base + (int64_t)__umul64hi(x, (uint64_t)n_nodes);
    }
}

__global__ void lp_concat_kernel(const int64_t* __restrict__ u, const int64_t* __restrict__ v, int64_t B,
                                 const int64_t* __restrict__ neg, int64_t n_neg, uint64_t* __restrict__ buf) {
    GSB_PDL_ENTRY();
    const int64_t n = 2 * B + n_neg;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        buf[i] = (uint64_t)(i < B ? u[i] : (i < 2 * B ? v[i - B] : neg[i - 2 * B]));
}

__global__ void lp_pos_kernel(const uint64_t* __restrict__ buf, int64_t B, int64_t n_neg,
                              const int64_t* __restrict__ seeds, const int64_t* __restrict__ n_seeds,
                              int32_t* __restrict__ iu, int32_t* __restrict__ iv, int32_t* __restrict__ ineg) {
    GSB_PDL_ENTRY();
    const int64_t n = 2 * B + n_neg;
    const int64_t ns = *n_seeds;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t x = (int64_t)buf[i];
        int64_t lo = 0, hi = ns;
        while (lo < hi) {
            int64_t m = (lo + hi) >> 1;
            if (seeds[m] < x) lo = m + 1; else hi = m;
        }
        if (i < B) iu[i] = (int32_t)lo;
        else if (i < 2 * B) iv[i - B] = (int32_t)lo;
        else ineg[i - 2 * B] = (int32_t)lo;
    }
}

// ------------------------------------------------------------------------------------
// DistMult + loss: warp per positive; lanes over the embedding (float4 chunks)
// ------------------------------------------------------------------------------------
constexpr int kMaxC4 = 4;   // d <= 512

__device__ __forceinline__ float warp_sum(float x) {
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    return x;
}

__device__ __forceinline__ float softplus(float x) { return x > 0.f ? x + log1pf(expf(-x)) : log1pf(expf(x)); }
__device__ __forceinline__ float sigm(float x) { return x >= 0.f ? 1.f / (1.f + expf(-x)) : expf(x) / (1.f + expf(x)); }

__global__ void __launch_bounds__(256) lp_score_kernel(const float* __restrict__ H, int d,
                                                       const int32_t* __restrict__ iu, const int32_t* __restrict__ iv,
                                                       const int32_t* __restrict__ ineg, int64_t B, int K,
                                                       int group, int mode, const float* __restrict__ rel, int kind,
                                                       const float* __restrict__ wpos,
                                                       float* __restrict__ scores, float* __restrict__ row_loss,
                                                       float* __restrict__ dH, float* __restrict__ drel) {
    GSB_PDL_ENTRY();
    extern __shared__ float s_drel[];
    const int lane = threadIdx.x & 31;
    const int d4 = d >> 2;
    for (int c = threadIdx.x; c < d; c += blockDim.x) s_drel[c] = 0.f;
    __syncthreads();
    float4 r[kMaxC4], dr[kMaxC4];
#pragma unroll
    for (int q = 0; q < kMaxC4; ++q) {
        int c = lane + 32 * q;
        r[q] = (c >= d4) ? make_float4(0.f, 0.f, 0.f, 0.f)
                         : (rel ? __ldg(reinterpret_cast<const float4*>(rel) + c) : make_float4(1.f, 1.f, 1.f, 1.f));
        dr[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const float invB = 1.f / (float)B;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < B; i += warps) {
        // row of negative j of positive i: sampled (mode 0, shared by `group` positives) or the
        // destination of another positive of the batch (mode 1, in-batch)
        const int64_t nb = (i / group) * K;
        auto neg_row = [&](int j) -> int64_t { return mode == 0 ? ineg[nb + j] : iv[j < i ? j : j + 1]; };
        const float* hu = H + (int64_t)iu[i] * d;
        const float* hv = H + (int64_t)iv[i] * d;
        float4 u[kMaxC4], ur[kMaxC4];
        float s0 = 0.f;
#pragma unroll
        for (int q = 0; q < kMaxC4; ++q) {
            int c = lane + 32 * q;
            u[q] = make_float4(0.f, 0.f, 0.f, 0.f);
            ur[q] = u[q];
            if (c < d4) {
                u[q] = reinterpret_cast<const float4*>(hu)[c];
                float4 v = reinterpret_cast<const float4*>(hv)[c];
                ur[q] = make_float4(u[q].x * r[q].x, u[q].y * r[q].y, u[q].z * r[q].z, u[q].w * r[q].w);
                s0 += ur[q].x * v.x + ur[q].y * v.y + ur[q].z * v.z + ur[q].w * v.w;
            }
        }
        s0 = warp_sum(s0);
        float* sc = scores + i * (K + 1);
        if (lane == 0) sc[0] = s0;
        // pass 1: negative scores, online max / sum-exp (contrastive) or BCE sum (CE)
        const float wi = (kind == 2) ? wpos[i] : 1.f;
        float mx = s0, se = 1.f, lsum = wi * softplus(-s0);
        for (int j = 0; j < K; ++j) {
            const float* hn = H + neg_row(j) * d;
            float s = 0.f;
#pragma unroll
            for (int q = 0; q < kMaxC4; ++q) {
                int c = lane + 32 * q;
                if (c < d4) {
                    float4 n = reinterpret_cast<const float4*>(hn)[c];
                    s += ur[q].x * n.x + ur[q].y * n.y + ur[q].z * n.z + ur[q].w * n.w;
                }
            }
            s = warp_sum(s);
            if (lane == 0) sc[1 + j] = s;
            if (s > mx) {
                se = se * expf(mx - s) + 1.f;
                mx = s;
            } else {
                se += expf(s - mx);
            }
            lsum += softplus(s);
        }
        const float lse = mx + logf(se);
        if (lane == 0) row_loss[i] = (kind == 0) ? (lse - s0) : lsum / (float)(K + 1);
        __syncwarp();
        // pass 2: gradients.  ds_j = dloss/dscore_j
        float4 du[kMaxC4];
        const float ds0 = (kind == 0) ? (expf(s0 - lse) - 1.f) * invB : wi * (sigm(s0) - 1.f) / (float)(K + 1) * invB;
        float* dv = dH + (int64_t)iv[i] * d;
#pragma unroll
        for (int q = 0; q < kMaxC4; ++q) {
            int c = lane + 32 * q;
            du[q] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (c < d4) {
                float4 v = reinterpret_cast<const float4*>(hv)[c];
                du[q] = make_float4(ds0 * r[q].x * v.x, ds0 * r[q].y * v.y, ds0 * r[q].z * v.z, ds0 * r[q].w * v.w);
                dr[q].x += ds0 * u[q].x * v.x; dr[q].y += ds0 * u[q].y * v.y;
                dr[q].z += ds0 * u[q].z * v.z; dr[q].w += ds0 * u[q].w * v.w;
                red_add_f4(dv + 4 * c, make_float4(ds0 * ur[q].x, ds0 * ur[q].y, ds0 * ur[q].z, ds0 * ur[q].w));
            }
        }
        for (int j = 0; j < K; ++j) {
            const float s = sc[1 + j];
            const float ds = (kind == 0) ? expf(s - lse) * invB : sigm(s) / (float)(K + 1) * invB;
            const int64_t row = neg_row(j);
            const float* hn = H + row * d;
            float* dn = dH + row * d;
#pragma unroll
            for (int q = 0; q < kMaxC4; ++q) {
                int c = lane + 32 * q;
                if (c < d4) {
                    float4 n = reinterpret_cast<const float4*>(hn)[c];
                    du[q].x += ds * r[q].x * n.x; du[q].y += ds * r[q].y * n.y;
                    du[q].z += ds * r[q].z * n.z; du[q].w += ds * r[q].w * n.w;
                    dr[q].x += ds * u[q].x * n.x; dr[q].y += ds * u[q].y * n.y;
                    dr[q].z += ds * u[q].z * n.z; dr[q].w += ds * u[q].w * n.w;
                    red_add_f4(dn + 4 * c, make_float4(ds * ur[q].x, ds * ur[q].y, ds * ur[q].z, ds * ur[q].w));
                }
            }
        }
        float* duo = dH + (int64_t)iu[i] * d;
#pragma unroll
        for (int q = 0; q < kMaxC4; ++q) {
            int c = lane + 32 * q;
            if (c < d4) red_add_f4(duo + 4 * c, du[q]);
        }
    }
#pragma unroll
    for (int q = 0; q < kMaxC4; ++q) {
        int c = lane + 32 * q;
        if (c < d4) {
            atomicAdd(&s_drel[4 * c + 0], dr[q].x);
            atomicAdd(&s_drel[4 * c + 1], dr[q].y);
            atomicAdd(&s_drel[4 * c + 2], dr[q].z);
            atomicAdd(&s_drel[4 * c + 3], dr[q].w);
        }
    }
    __syncthreads();
    if (rel)
        for (int c = threadIdx.x; c < d; c += blockDim.x) atomicAdd(drel + c, s_drel[c]);
}

// ------------------------------------------------------------------------------------
// Joint negatives (group == K <= 32): one CTA per group of K positives that share K
// negatives.  The negatives' rows are staged in shared memory once per group (instead of once
// per positive), lane j of a positive's warp scores negative j against the staged u*r row, and
// the negatives' gradients dH[neg_j] += sum_i ds_ij (u_i * r) are reduced over the group in
// shared memory and added once per group (instead of one red.add per positive and negative).
// ------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) lp_group_kernel(const float* __restrict__ H, int d,
                                                       const int32_t* __restrict__ iu, const int32_t* __restrict__ iv,
                                                       const int32_t* __restrict__ ineg, int64_t B, int K,
                                                       const float* __restrict__ rel, int kind,
                                                       const float* __restrict__ wpos, float* __restrict__ scores,
                                                       float* __restrict__ row_loss, float* __restrict__ dH,
                                                       float* __restrict__ drel) {
    GSB_PDL_ENTRY();
    extern __shared__ float sm[];
    const int d4 = d >> 2, ldn = d + 4;
    float* s_neg = sm;                      // [K][ldn] negative rows
    float* s_ur = s_neg + K * ldn;          // [K][ldn] u*r of the group's positives
    float* s_ds = s_ur + K * ldn;           // [K][32]  dloss / dscore(positive p, negative j)
    float* s_drel = s_ds + K * 32;          // [d]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    for (int c = tid; c < d; c += blockDim.x) s_drel[c] = 0.f;
    float4 r[kMaxC4], dr[kMaxC4];
#pragma unroll
    for (int q = 0; q < kMaxC4; ++q) {
        const int c = lane + 32 * q;
        r[q] = (c >= d4) ? make_float4(0.f, 0.f, 0.f, 0.f)
                         : (rel ? __ldg(reinterpret_cast<const float4*>(rel) + c) : make_float4(1.f, 1.f, 1.f, 1.f));
        dr[q] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const float invB = 1.f / (float)B;
    const int64_t G = (B + K - 1) / K;
    for (int64_t g = blockIdx.x; g < G; g += gridDim.x) {
        const int64_t i0 = g * K;
        const int np = (int)min((int64_t)K, B - i0);
        __syncthreads();       // the previous group's readers of s_neg / s_ur / s_ds are done
        for (int x = tid; x < K * d4; x += blockDim.x) {
            const int j = x / d4, c = x - j * d4;
            *reinterpret_cast<float4*>(s_neg + j * ldn + 4 * c) =
                __ldg(reinterpret_cast<const float4*>(H + (int64_t)ineg[i0 + j] * d) + c);
        }
        __syncthreads();
        for (int p = warp; p < np; p += nwarps) {
            const int64_t i = i0 + p;
            const float* hu = H + (int64_t)iu[i] * d;
            const float* hv = H + (int64_t)iv[i] * d;
            float4 u[kMaxC4], ur[kMaxC4], v[kMaxC4];
            float s0 = 0.f;
#pragma unroll
            for (int q = 0; q < kMaxC4; ++q) {
                const int c = lane + 32 * q;
                u[q] = v[q] = ur[q] = make_float4(0.f, 0.f, 0.f, 0.f);
                if (c < d4) {
                    u[q] = reinterpret_cast<const float4*>(hu)[c];
                    v[q] = reinterpret_cast<const float4*>(hv)[c];
                    ur[q] = make_float4(u[q].x * r[q].x, u[q].y * r[q].y, u[q].z * r[q].z, u[q].w * r[q].w);
                    s0 += ur[q].x * v[q].x + ur[q].y * v[q].y + ur[q].z * v[q].z + ur[q].w * v[q].w;
                    *reinterpret_cast<float4*>(s_ur + p * ldn + 4 * c) = ur[q];
                }
            }
            s0 = warp_sum(s0);
            __syncwarp();
            // lane j: score of negative j (rows padded to ldn: lanes hit distinct banks)
            float sj = 0.f;
            if (lane < K) {
                const float4* a = reinterpret_cast<const float4*>(s_ur + p * ldn);
                const float4* b = reinterpret_cast<const float4*>(s_neg + lane * ldn);
                for (int c = 0; c < d4; ++c) {
                    const float4 x = a[c], y = b[c];
                    sj += x.x * y.x + x.y * y.y + x.z * y.z + x.w * y.w;
                }
            }
            float* sc = scores + i * (K + 1);
            if (lane == 0) sc[0] = s0;
            if (lane < K) sc[1 + lane] = sj;
            float mx = (lane < K) ? fmaxf(sj, s0) : s0;
            for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
            const float se = expf(s0 - mx) + warp_sum(lane < K ? expf(sj - mx) : 0.f);
            const float lse = mx + logf(se);
            const float wi = (kind == 2) ? wpos[i] : 1.f;
            const float lsum = wi * softplus(-s0) + warp_sum(lane < K ? softplus(sj) : 0.f);
            if (lane == 0) row_loss[i] = (kind == 0) ? (lse - s0) : lsum / (float)(K + 1);
            const float ds0 =
                (kind == 0) ? (expf(s0 - lse) - 1.f) * invB : wi * (sigm(s0) - 1.f) / (float)(K + 1) * invB;
            const float dsj = (lane < K) ? ((kind == 0) ? expf(sj - lse) * invB : sigm(sj) / (float)(K + 1) * invB) : 0.f;
            s_ds[p * 32 + lane] = dsj;
            float4 du[kMaxC4];
#pragma unroll
            for (int q = 0; q < kMaxC4; ++q) {
                du[q] = make_float4(ds0 * r[q].x * v[q].x, ds0 * r[q].y * v[q].y, ds0 * r[q].z * v[q].z,
                                    ds0 * r[q].w * v[q].w);
                dr[q].x += ds0 * u[q].x * v[q].x; dr[q].y += ds0 * u[q].y * v[q].y;
                dr[q].z += ds0 * u[q].z * v[q].z; dr[q].w += ds0 * u[q].w * v[q].w;
            }
            for (int j = 0; j < K; ++j) {
                const float ds = __shfl_sync(0xffffffffu, dsj, j);
#pragma unroll
                for (int q = 0; q < kMaxC4; ++q) {
                    const int c = lane + 32 * q;
                    if (c < d4) {
                        const float4 n = *reinterpret_cast<const float4*>(s_neg + j * ldn + 4 * c);
                        du[q].x += ds * r[q].x * n.x; du[q].y += ds * r[q].y * n.y;
                        du[q].z += ds * r[q].z * n.z; du[q].w += ds * r[q].w * n.w;
                        dr[q].x += ds * u[q].x * n.x; dr[q].y += ds * u[q].y * n.y;
                        dr[q].z += ds * u[q].z * n.z; dr[q].w += ds * u[q].w * n.w;
                    }
                }
            }
            float* duo = dH + (int64_t)iu[i] * d;
            float* dvo = dH + (int64_t)iv[i] * d;
#pragma unroll
            for (int q = 0; q < kMaxC4; ++q) {
                const int c = lane + 32 * q;
                if (c < d4) {
                    red_add_f4(duo + 4 * c, du[q]);
                    red_add_f4(dvo + 4 * c, make_float4(ds0 * ur[q].x, ds0 * ur[q].y, ds0 * ur[q].z, ds0 * ur[q].w));
                }
            }
        }
        __syncthreads();
        // negatives: dH[neg_j] += sum over the group's positives p of ds[p][j] * (u_p * r)
        for (int x = tid; x < K * d4; x += blockDim.x) {
            const int j = x / d4, c = x - j * d4;
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int p = 0; p < np; ++p) {
                const float w = s_ds[p * 32 + j];
                const float4 y = *reinterpret_cast<const float4*>(s_ur + p * ldn + 4 * c);
                acc.x += w * y.x; acc.y += w * y.y; acc.z += w * y.z; acc.w += w * y.w;
            }
            red_add_f4(dH + (int64_t)ineg[i0 + j] * d + 4 * c, acc);
        }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < kMaxC4; ++q) {
        const int c = lane + 32 * q;
        if (c < d4) {
            atomicAdd(&s_drel[4 * c + 0], dr[q].x);
            atomicAdd(&s_drel[4 * c + 1], dr[q].y);
            atomicAdd(&s_drel[4 * c + 2], dr[q].z);
            atomicAdd(&s_drel[4 * c + 3], dr[q].w);
        }
    }
    __syncthreads();
    if (rel)
        for (int c = tid; c < d; c += blockDim.x) atomicAdd(drel + c, s_drel[c]);
}

__global__ void __launch_bounds__(1024) lp_mean_kernel(const float* __restrict__ x, int64_t n, float* __restrict__ out) {
    GSB_PDL_ENTRY();
    __shared__ float sm[32];
    float s = 0.f;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += x[i];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = (threadIdx.x < (blockDim.x >> 5)) ? sm[threadIdx.x] : 0.f;
        s = warp_sum(s);
        if (threadIdx.x == 0) *out = s / (float)n;
    }
}

// MRR (R-mrr): warp per positive, lanes over its K negatives; rank = 1 + #higher +
// #equal / 2 (counts exact, compared in the scores' own fp32), rr = 1 / rank
__global__ void __launch_bounds__(256) lp_rr_kernel(const float* __restrict__ scores, int64_t ld, int64_t B, int K,
                                                    float* __restrict__ rr) {
    GSB_PDL_ENTRY();
    const int lane = threadIdx.x & 31;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < B; i += warps) {
        const float* row = scores + i * ld;
        const float pos = row[0];
        int gt = 0, eq = 0;
        for (int j = 1 + lane; j <= K; j += 32) {
            const float x = row[j];
            gt += x > pos;
            eq += x == pos;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            gt += __shfl_xor_sync(0xffffffffu, gt, o);
            eq += __shfl_xor_sync(0xffffffffu, eq, o);
        }
        if (lane == 0) rr[i] = 1.f / (1.f + (float)gt + 0.5f * (float)eq);
    }
}


// ------------------------------------------------------------------------------------
// In-batch negatives as dense contractions (App. A.2.1): with U = H[iu], V = H[iv]
// and Ur = U o r, every score of the batch is S = Ur V^T (B x B; S_ii the positive, row i's
// other entries its B-1 negatives in batch order).  Backward: M = dS V, dU = M o r,
// drel = sum_i U_i o M_i, dV = dS^T Ur.  The three products run on the tcgen05 3xTF32 GEMM
// (gsb_gemm); these kernels do the row-wise loss and the gathers / scatters.
// ------------------------------------------------------------------------------------
__global__ void ib_gather_kernel(const float* __restrict__ H, int d, const int32_t* __restrict__ iu,
                                 const int32_t* __restrict__ iv, int64_t B, const float* __restrict__ rel,
                                 float* __restrict__ U, float* __restrict__ V, float* __restrict__ Ur) {
    GSB_PDL_ENTRY();
    const int d4 = d >> 2;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < B * d4; x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = x / d4;
        const int c = (int)(x % d4);
        const float4 u = reinterpret_cast<const float4*>(H + (int64_t)iu[i] * d)[c];
        const float4 v = reinterpret_cast<const float4*>(H + (int64_t)iv[i] * d)[c];
        const float4 r = rel ? reinterpret_cast<const float4*>(rel)[c] : make_float4(1.f, 1.f, 1.f, 1.f);
        reinterpret_cast<float4*>(U)[x] = u;
        reinterpret_cast<float4*>(V)[x] = v;
        reinterpret_cast<float4*>(Ur)[x] = make_float4(u.x * r.x, u.y * r.y, u.z * r.z, u.w * r.w);
    }
}

// warp per row i of S: loss_i, scores row [S_ii, S_i0 .. (skipping i) .. S_i,B-1], dS row in place
__global__ void __launch_bounds__(256) ib_rows_kernel(float* __restrict__ S, int64_t B, int kind,
                                                      const float* __restrict__ wpos, float* __restrict__ scores,
                                                      float* __restrict__ row_loss) {
    GSB_PDL_ENTRY();
    const int lane = threadIdx.x & 31;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const float invB = 1.f / (float)B;
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < B; i += warps) {
        float* row = S + i * B;
        float* sc = scores + i * B;
        const float s0 = row[i];
        float mx = -INFINITY, lsum = 0.f;
        const float wi = (kind == 2) ? wpos[i] : 1.f;
        for (int64_t j = lane; j < B; j += 32) {
            const float x = row[j];
            mx = fmaxf(mx, x);
            lsum += (j == i) ? wi * softplus(-x) : softplus(x);
            sc[j < i ? j + 1 : (j == i ? 0 : j)] = x;
        }
        for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        float se = 0.f;
        for (int64_t j = lane; j < B; j += 32) se += expf(row[j] - mx);
        se = warp_sum(se);
        lsum = warp_sum(lsum);
        const float lse = mx + logf(se);
        if (lane == 0) row_loss[i] = (kind == 0) ? (lse - s0) : lsum / (float)B;
        for (int64_t j = lane; j < B; j += 32) {
            const float x = row[j];
            float g;
            if (kind == 0) g = (expf(x - lse) - (j == i ? 1.f : 0.f)) * invB;
            else g = (j == i ? wi * (sigm(x) - 1.f) : sigm(x)) / (float)B * invB;
            row[j] = g;
        }
    }
}

// dU = M o r scattered to dH[iu], dV scattered to dH[iv], drel = sum_i U_i o M_i
__global__ void __launch_bounds__(256) ib_finish_kernel(const float* __restrict__ U, const float* __restrict__ M,
                                                        const float* __restrict__ dV, const int32_t* __restrict__ iu,
                                                        const int32_t* __restrict__ iv, int64_t B, int d,
                                                        const float* __restrict__ rel, float* __restrict__ dH,
                                                        float* __restrict__ drel) {
    GSB_PDL_ENTRY();
    extern __shared__ float s_dr[];
    for (int c = threadIdx.x; c < d; c += blockDim.x) s_dr[c] = 0.f;
    __syncthreads();
    const int d4 = d >> 2;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < B * d4; x += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = x / d4;
        const int c = (int)(x % d4);
        const float4 m = reinterpret_cast<const float4*>(M)[x];
        const float4 r = rel ? reinterpret_cast<const float4*>(rel)[c] : make_float4(1.f, 1.f, 1.f, 1.f);
        red_add_f4(dH + (int64_t)iu[i] * d + 4 * c, make_float4(m.x * r.x, m.y * r.y, m.z * r.z, m.w * r.w));
        red_add_f4(dH + (int64_t)iv[i] * d + 4 * c, reinterpret_cast<const float4*>(dV)[x]);
        if (rel) {
            const float4 u = reinterpret_cast<const float4*>(U)[x];
            atomicAdd(&s_dr[4 * c + 0], u.x * m.x);
            atomicAdd(&s_dr[4 * c + 1], u.y * m.y);
            atomicAdd(&s_dr[4 * c + 2], u.z * m.z);
            atomicAdd(&s_dr[4 * c + 3], u.w * m.w);
        }
    }
    __syncthreads();
    if (rel)
        for (int c = threadIdx.x; c < d; c += blockDim.x) atomicAdd(drel + c, s_dr[c]);
}

static bool inbatch_gemm_ok(int64_t B) { return B % 32 == 0 && B >= 32; }

static size_t lp_cub_bytes(int64_t n) {
    size_t a = 0, b = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, a, (const uint64_t*)nullptr, (uint64_t*)nullptr, (int64_t)n, 0, 64);
    cub::DeviceSelect::Unique(nullptr, b, (const uint64_t*)nullptr, (uint64_t*)nullptr, (int64_t*)nullptr, (int64_t)n);
    return std::max(a, b);
}

}  // namespace gsb

using namespace gsb;

extern "C" {

gsb_status gsb_joint_negatives(int64_t n_pos, int32_t K, int64_t n_dst_nodes, int64_t gid_base, uint64_t rng_seed,
                               uint32_t step, const uint32_t* step_dev, int64_t group_base, int64_t* neg,
                               void* stream) {
    GSB_CHECK_ARG(neg && n_pos >= 1 && K >= 1 && K <= 0xFFFF && n_dst_nodes >= 1, "bad argument");
    const int64_t total = ceil_div(n_pos, K) * K;
    GSB_LAUNCH("joint_negatives", joint_neg_kernel, grid_for(total, 256, kNumSMs * 4), 256, 0, (cudaStream_t)stream,
               total, K, n_dst_nodes, gid_base, rng_seed, step, step_dev, group_base, neg, 0xFFF00000u);
    return GSB_OK;
}

gsb_status gsb_uniform_negatives(int64_t n_pos, int32_t K, int64_t n_dst_nodes, int64_t gid_base, uint64_t rng_seed,
                                 uint32_t step, const uint32_t* step_dev, int64_t pos_base, int64_t* neg,
                                 void* stream) {
    GSB_CHECK_ARG(neg && n_pos >= 1 && K >= 1 && K <= 0xFFFF && n_dst_nodes >= 1, "bad argument");
    const int64_t total = n_pos * K;
    GSB_LAUNCH("uniform_negatives", joint_neg_kernel, grid_for(total, 256, kNumSMs * 4), 256, 0, (cudaStream_t)stream,
               total, K, n_dst_nodes, gid_base, rng_seed, step, step_dev, pos_base, neg, 0xFFE00000u);
    return GSB_OK;
}

gsb_status gsb_lp_seeds_bytes(int64_t B, int64_t n_neg, size_t* bytes) {
    GSB_CHECK_ARG(bytes && B >= 1 && n_neg >= 0, "bad argument");
    const int64_t n = 2 * B + n_neg;
    *bytes = 2 * align_up(sizeof(uint64_t) * n) + align_up(lp_cub_bytes(n));
    return GSB_OK;
}

gsb_status gsb_lp_seeds(const int64_t* u, const int64_t* v, int64_t B, const int64_t* neg, int64_t n_neg,
                        int64_t* seeds, int64_t* n_seeds_dev, int32_t* iu, int32_t* iv, int32_t* ineg, void* ws,
                        size_t ws_bytes, void* stream) {
    GSB_CHECK_ARG(u && v && seeds && n_seeds_dev && iu && iv && ws && B >= 1 && n_neg >= 0, "null argument");
    GSB_CHECK_ARG(n_neg == 0 || (neg && ineg), "null negatives");
    size_t need = 0;
    gsb_lp_seeds_bytes(B, n_neg, &need);
    if (ws_bytes < need) {
        set_error("lp_seeds workspace %zu < %zu", ws_bytes, need);
        return GSB_EWORKSPACE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n = 2 * B + n_neg;
    uint64_t* buf = (uint64_t*)ws;
    uint64_t* sorted = (uint64_t*)((char*)ws + align_up(sizeof(uint64_t) * n));
    void* tmp = (char*)ws + 2 * align_up(sizeof(uint64_t) * n);
    size_t tb = lp_cub_bytes(n);
    GSB_LAUNCH("lp_concat", lp_concat_kernel, grid_for(n, 256, kNumSMs * 4), 256, 0, s, u, v, B, neg, n_neg, buf);
    GSB_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tb, buf, sorted, (int64_t)n, 0, 40, s));
    count_launch(12);
    tb = lp_cub_bytes(n);
    GSB_CUDA(cub::DeviceSelect::Unique(tmp, tb, sorted, (uint64_t*)seeds, n_seeds_dev, (int64_t)n, s));
    count_launch(2);
    GSB_LAUNCH("lp_positions", lp_pos_kernel, grid_for(n, 256, kNumSMs * 4), 256, 0, s, buf, B, n_neg, seeds,
               n_seeds_dev, iu, iv, ineg);
    return GSB_OK;
}

gsb_status gsb_lp_score_ws_bytes(int64_t B, int32_t d, int32_t neg_mode, size_t* bytes) {
    GSB_CHECK_ARG(bytes && B >= 1 && d > 0, "bad argument");
    *bytes = (neg_mode == 1 && inbatch_gemm_ok(B))
                 ? sizeof(float) * (size_t)(5 * B * (int64_t)d + B * B) : 0;
    return GSB_OK;
}

gsb_status gsb_lp_score_ex(const float* H, int64_t n_rows_cap, int32_t d, const int32_t* iu, const int32_t* iv,
                           const int32_t* ineg, int64_t B, int32_t K, int32_t group, int32_t neg_mode,
                           const float* rel, int32_t loss_kind, const float* w, float* scores, float* row_loss_ws,
                           float* loss, float* dH, float* drel, void* ws, size_t ws_bytes, void* stream) {
    GSB_CHECK_ARG(H && iu && iv && scores && row_loss_ws && loss && dH, "null argument");
    GSB_CHECK_ARG(d > 0 && d % 4 == 0 && d <= 4 * 32 * kMaxC4, "d %d must be a multiple of 4 and <= %d", d,
                  4 * 32 * kMaxC4);
    GSB_CHECK_ARG(B >= 1 && K >= 1 && loss_kind >= 0 && loss_kind <= 2, "bad B/K/loss_kind");
    GSB_CHECK_ARG(neg_mode == 0 || neg_mode == 1, "neg_mode must be 0 (sampled) or 1 (in-batch)");
    GSB_CHECK_ARG(neg_mode == 1 || (ineg && group >= 1), "sampled negatives need ineg and group >= 1");
    GSB_CHECK_ARG(neg_mode == 0 || K == B - 1, "in-batch negatives need K = B - 1 (K %d, B %lld)", K, (long long)B);
    GSB_CHECK_ARG(!rel || drel, "DistMult needs drel");
    GSB_CHECK_ARG(loss_kind != 2 || w, "weighted cross entropy needs w");
    size_t need = 0;
    gsb_lp_score_ws_bytes(B, d, neg_mode, &need);
    if (ws_bytes < need || (need && !ws)) {
        set_error("lp_score workspace %zu < %zu", ws_bytes, need);
        return GSB_EWORKSPACE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    GSB_CUDA(cudaMemsetAsync(dH, 0, sizeof(float) * (size_t)n_rows_cap * d, s));
    if (rel) GSB_CUDA(cudaMemsetAsync(drel, 0, sizeof(float) * (size_t)d, s));
    if (need) {   // in-batch on the tensor cores
        float* U = (float*)ws;
        float* V = U + B * d;
        float* Ur = V + B * d;
        float* M = Ur + B * d;
        float* dV = M + B * d;
        float* S = dV + B * d;
        const int64_t n4 = B * (d / 4);
        GSB_LAUNCH("lp_ib_gather", ib_gather_kernel, grid_for(n4, 256, kNumSMs * 8), 256, 0, s, H, d, iu, iv, B, rel,
                   U, V, Ur);
        gsb_status st = gsb_gemm(1, Ur, d, V, d, B, d, (int32_t)B, S, B, s);          // S = Ur V^T
        if (st != GSB_OK) return st;
        GSB_LAUNCH("lp_ib_rows", ib_rows_kernel, grid_for(B * 32, 256, kNumSMs * 8), 256, 0, s, S, B, loss_kind, w,
                   scores, row_loss_ws);
        st = gsb_gemm(0, S, B, V, d, B, d, (int32_t)B, M, d, s);                     // M = dS V
        if (st != GSB_OK) return st;
        GSB_CUDA(cudaMemsetAsync(dV, 0, sizeof(float) * (size_t)(B * d), s));
        st = gsb_gemm(2, S, B, Ur, d, B, d, (int32_t)B, dV, d, s);                   // dV = dS^T Ur
        if (st != GSB_OK) return st;
        GSB_LAUNCH("lp_ib_finish", ib_finish_kernel, grid_for(n4, 256, kNumSMs * 4), 256, sizeof(float) * d, s, U, M,
                   dV, iu, iv, B, d, rel, dH, drel);
    } else if (neg_mode == 0 && group == K && K <= 32 && !getenv("GSB_LP_WARP")) {
        // joint negatives: one CTA per group (GSB_LP_WARP=1: the warp-per-positive kernel, A/B)
        const size_t smem = sizeof(float) * (size_t)(2 * K * (d + 4) + K * 32 + d);
        static size_t smem_set = 0;
        if (smem > 48 * 1024 && smem > smem_set) {
            GSB_CUDA(cudaFuncSetAttribute(lp_group_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
            smem_set = smem;
        }
        const int64_t G = (B + K - 1) / K;
        GSB_LAUNCH("lp_score", lp_group_kernel, (int)std::min<int64_t>(G, kNumSMs * 8), 256, smem, s, H, d, iu, iv,
                   ineg, B, K, rel, loss_kind, w, scores, row_loss_ws, dH, drel);
    } else {
        GSB_LAUNCH("lp_score", lp_score_kernel, grid_for(B * 32, 256, kNumSMs * 4), 256, sizeof(float) * d, s, H, d,
                   iu, iv, ineg, B, K, neg_mode == 0 ? group : 1, neg_mode, rel, loss_kind, w, scores, row_loss_ws,
                   dH, drel);
    }
    GSB_LAUNCH("lp_mean", lp_mean_kernel, 1, 1024, 0, s, row_loss_ws, B, loss);
    return GSB_OK;
}

gsb_status gsb_lp_mrr(const float* scores, int64_t ld, int64_t B, int32_t K, float* rr, float* mrr, void* stream) {
    GSB_CHECK_ARG(scores && rr && mrr, "null argument");
    GSB_CHECK_ARG(B >= 1 && K >= 1 && ld >= (int64_t)K + 1, "B %lld, K %d, ld %lld", (long long)B, K, (long long)ld);
    cudaStream_t s = (cudaStream_t)stream;
    GSB_LAUNCH("lp_rr", lp_rr_kernel, grid_for(B * 32, 256, kNumSMs * 8), 256, 0, s, scores, ld, B, (int)K, rr);
    GSB_LAUNCH("lp_mean", lp_mean_kernel, 1, 1024, 0, s, rr, B, mrr);
    return GSB_OK;
}

gsb_status gsb_lp_score(const float* H, int64_t n_rows_cap, int32_t d, const int32_t* iu, const int32_t* iv,
                        const int32_t* ineg, int64_t B, int32_t K, const float* rel, int32_t loss_kind, float* scores,
                        float* row_loss_ws, float* loss, float* dH, float* drel, void* stream) {
    GSB_CHECK_ARG(rel && ineg && (loss_kind == 0 || loss_kind == 1), "gsb_lp_score: DistMult + joint negatives");
    return gsb_lp_score_ex(H, n_rows_cap, d, iu, iv, ineg, B, K, K, 0, rel, loss_kind, nullptr, scores, row_loss_ws,
                           loss, dH, drel, nullptr, 0, stream);
}

}  // extern "C"
