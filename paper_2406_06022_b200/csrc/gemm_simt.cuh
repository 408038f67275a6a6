// gemm_simt.cuh -- grouped fp32 FFMA GEMMs for the RGCN layer (round-1 parity path).
//
// The M (row) dimension is partitioned into groups = destination node types; group t
// multiplies its rows by a per-group stack of K-slots, slot s using weight matrix
// W[slot_w[t][s]] (row-major [d_in][ldw]).  Three shapes:
//   NN : C[r, n]          = act( sum_s A[r, s*d_in:(s+1)*d_in] @ W[slot] + bias )
//   NT : C[r, s*d_in + k] = sum_n dZ[r, n] * W[slot][k][n]        (dA = dZ W^T)
//   TN : dW[slot][k][n]  += sum_r A[r, s*d_in + k] * dZ[r, n]      (dW = A^T dZ), db += sum_r dZ
// dZ = dh * 1[h > 0] is formed on load when relu is set (h = layer output).
// CTA tile 64 x 128, k-tile 32, 256 threads, 4 x 8 outputs per thread, register prefetch.
#pragma once
#include "gsb_internal.cuh"

namespace gsb {

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

constexpr int BM = 64, BN = 128, BK = 32, NT = 256;
constexpr int APAD = 4;

// ------------------------------------------------------------------------------------
// the 4x8 micro-kernel over one staged k-tile
// ------------------------------------------------------------------------------------
__device__ __forceinline__ void mma_tile(const float (*As)[BM + APAD], const float (*Bs)[BN], float acc[4][8], int tx,
                                         int ty) {
#pragma unroll 8
    for (int k = 0; k < BK; ++k) {
        float4 a = *reinterpret_cast<const float4*>(&As[k][ty * 4]);
        float4 b0 = *reinterpret_cast<const float4*>(&Bs[k][tx * 4]);
        float4 b1 = *reinterpret_cast<const float4*>(&Bs[k][64 + tx * 4]);
        float av[4] = {a.x, a.y, a.z, a.w};
        float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
}

__device__ __forceinline__ int out_col(int tx, int j) { return (j < 4) ? tx * 4 + j : 64 + tx * 4 + (j - 4); }

// ------------------------------------------------------------------------------------
// NN: fwd layer GEMM and decoder logits
// ------------------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) gemm_nn_kernel(RowGroups rg, const float* __restrict__ A, int64_t lda,
                                                     const float* __restrict__ W, int d_in, int N, int64_t ldw,
                                                     int64_t wslot_stride, const float* __restrict__ bias, int relu,
                                                     float* __restrict__ C, int64_t ldc) {
    GSB_PDL_ENTRY();
    __shared__ __align__(16) float As[BK][BM + APAD];
    __shared__ __align__(16) float Bs[BK][BN];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int ntn = (N + BN - 1) / BN;
    // count tiles
    int64_t total = 0;
    for (int t = 0; t < rg.G; ++t) {
        int64_t r0, r1;
        group_rows(rg, t, r0, r1);
        total += ((r1 - r0 + BM - 1) / BM) * ntn;
    }
    for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
        int t = 0;
        int64_t rem = tile, r0 = 0, r1 = 0;
        for (;; ++t) {
            group_rows(rg, t, r0, r1);
            int64_t nt = ((r1 - r0 + BM - 1) / BM) * ntn;
            if (rem < nt) break;
            rem -= nt;
        }
        const int64_t row0 = r0 + (rem / ntn) * BM;
        const int n0 = (int)(rem % ntn) * BN;
        float acc[4][8];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
        const int KS = rg.ks[t];
        const int ktiles = KS * (d_in / BK);
        // A load mapping: 2048 elems, 8 per thread: row = (tid>>5) + 8*i, k = tid & 31
        const int ak = tid & 31, ar = tid >> 5;
        float ra[8], rb[16];
        auto load = [&](int kt) {
            const int s = kt / (d_in / BK);
            const int kk = (kt - s * (d_in / BK)) * BK;
            const int64_t acol = (int64_t)s * d_in + kk + ak;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                int64_t row = row0 + ar + 8 * i;
                ra[i] = (row < r1) ? __ldg(A + row * lda + acol) : 0.f;
            }
            const float* Bp = W + (int64_t)rg.slot_w[t][s] * wslot_stride + (int64_t)kk * ldw;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                int idx = tid + i * NT;  // 0..4095
                int k = idx >> 7, n = idx & 127;
                rb[i] = (n0 + n < N) ? __ldg(Bp + (int64_t)k * ldw + n0 + n) : 0.f;
            }
        };
        auto store = [&]() {
#pragma unroll
            for (int i = 0; i < 8; ++i) As[ak][ar + 8 * i] = ra[i];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                int idx = tid + i * NT;
                Bs[idx >> 7][idx & 127] = rb[i];
            }
        };
        load(0);
        for (int kt = 0; kt < ktiles; ++kt) {
            __syncthreads();
            store();
            __syncthreads();
            if (kt + 1 < ktiles) load(kt + 1);
            mma_tile(As, Bs, acc, tx, ty);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            int64_t row = row0 + ty * 4 + i;
            if (row >= r1) continue;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                int n = n0 + out_col(tx, j);
                if (n < N) {
                    float v = acc[i][j] + (bias ? __ldg(bias + n) : 0.f);
                    if (relu) v = fmaxf(v, 0.f);
                    C[row * ldc + n] = v;
                }
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------------
// NT: dA[r, s*d_in + k] = sum_n dZ[r, n] W[slot][k][n]   (reduction over n < N)
// ------------------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) gemm_nt_kernel(RowGroups rg, const float* __restrict__ dH,
                                                     const float* __restrict__ H, int relu, int64_t ldh,
                                                     const float* __restrict__ W, int d_in, int N, int64_t ldw,
                                                     int64_t wslot_stride, float* __restrict__ C, int64_t ldc) {
    GSB_PDL_ENTRY();
    __shared__ __align__(16) float As[BK][BM + APAD];
    __shared__ __align__(16) float Bs[BK][BN];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int ntk = (d_in + BN - 1) / BN;  // column tiles per slot
    int64_t total = 0;
    for (int t = 0; t < rg.G; ++t) {
        int64_t r0, r1;
        group_rows(rg, t, r0, r1);
        total += ((r1 - r0 + BM - 1) / BM) * ntk * rg.ks[t];
    }
    for (int64_t tile = blockIdx.x; tile < total; tile += gridDim.x) {
        int t = 0;
        int64_t rem = tile, r0 = 0, r1 = 0;
        for (;; ++t) {
            group_rows(rg, t, r0, r1);
            int64_t nt = ((r1 - r0 + BM - 1) / BM) * ntk * rg.ks[t];
            if (rem < nt) break;
            rem -= nt;
        }
        const int per_row_tile = ntk * rg.ks[t];
        const int64_t row0 = r0 + (rem / per_row_tile) * BM;
        const int cidx = (int)(rem % per_row_tile);
        const int s = cidx / ntk;
        const int k0 = (cidx % ntk) * BN;
        const float* Wp = W + (int64_t)rg.slot_w[t][s] * wslot_stride;
        float acc[4][8];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
        const int ktiles = (N + BK - 1) / BK;
        const int ak = tid & 31, ar = tid >> 5;
        float ra[8], rb[16];
        auto load = [&](int kt) {
            const int nn = kt * BK + ak;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                int64_t row = row0 + ar + 8 * i;
                float v = 0.f;
                if (row < r1 && nn < N) {
                    v = __ldg(dH + row * ldh + nn);
                    if (relu && __ldg(H + row * ldh + nn) <= 0.f) v = 0.f;
                }
                ra[i] = v;
            }
            // Bs[n][k] = W[k0 + k][kt*BK + n]: thread reads along n (contiguous)
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                int idx = tid + i * NT;  // 0..4095 -> k = idx >> 5 (0..127), n = idx & 31
                int k = idx >> 5, n = idx & 31;
                int nn2 = kt * BK + n;
                rb[i] = (k0 + k < d_in && nn2 < N) ? __ldg(Wp + (int64_t)(k0 + k) * ldw + nn2) : 0.f;
            }
        };
        auto store = [&]() {
#pragma unroll
            for (int i = 0; i < 8; ++i) As[ak][ar + 8 * i] = ra[i];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                int idx = tid + i * NT;
                Bs[idx & 31][idx >> 5] = rb[i];
            }
        };
        load(0);
        for (int kt = 0; kt < ktiles; ++kt) {
            __syncthreads();
            store();
            __syncthreads();
            if (kt + 1 < ktiles) load(kt + 1);
            mma_tile(As, Bs, acc, tx, ty);
        }
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            int64_t row = row0 + ty * 4 + i;
            if (row >= r1) continue;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                int k = k0 + out_col(tx, j);
                if (k < d_in) C[row * ldc + (int64_t)s * d_in + k] = acc[i][j];
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------------------
// TN: dW[slot][k][n] += sum_{r in chunk} A[r, s*d_in + k] dZ[r, n] ; db[n] += sum_r dZ[r, n]
// ------------------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) gemm_tn_kernel(RowGroups rg, const float* __restrict__ A, int64_t lda,
                                                     const float* __restrict__ dH, const float* __restrict__ H,
                                                     int relu, int64_t ldh, int d_in, int N, int rows_per_chunk,
                                                     float* __restrict__ dW, int64_t ldw, int64_t wslot_stride,
                                                     float* __restrict__ db) {
    GSB_PDL_ENTRY();
    __shared__ __align__(16) float As[BK][BM + APAD];
    __shared__ __align__(16) float Bs[BK][BN];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    const int nkt = (d_in + BM - 1) / BM;   // output row tiles over k
    const int nnt = (N + BN - 1) / BN;      // output col tiles over n
    int64_t total = 0;
    for (int t = 0; t < rg.G; ++t) {
        int64_t r0, r1;
        group_rows(rg, t, r0, r1);
        total += ((r1 - r0 + rows_per_chunk - 1) / rows_per_chunk) * rg.ks[t] * nkt * nnt;
    }
    for (int64_t item = blockIdx.x; item < total; item += gridDim.x) {
        int t = 0;
        int64_t rem = item, r0 = 0, r1 = 0;
        for (;; ++t) {
            group_rows(rg, t, r0, r1);
            int64_t nt = ((r1 - r0 + rows_per_chunk - 1) / rows_per_chunk) * rg.ks[t] * nkt * nnt;
            if (rem < nt) break;
            rem -= nt;
        }
        const int per_chunk = rg.ks[t] * nkt * nnt;
        const int64_t c0 = r0 + (rem / per_chunk) * rows_per_chunk;
        const int64_t c1 = min(r1, c0 + rows_per_chunk);
        int q = (int)(rem % per_chunk);
        const int s = q / (nkt * nnt);
        q -= s * nkt * nnt;
        const int k0 = (q / nnt) * BM;
        const int n0 = (q % nnt) * BN;
        const bool do_db = db && (s == rg.ks[t] - 1) && k0 == 0;  // self slot exists once per group
        float acc[4][8];
        float cs[8];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
#pragma unroll
        for (int j = 0; j < 8; ++j) cs[j] = 0.f;
        const int64_t acol0 = (int64_t)s * d_in + k0;
        float ra[8], rb[16];
        const int ntiles = (int)((c1 - c0 + BK - 1) / BK);
        auto load = [&](int it) {
            const int64_t rbase = c0 + (int64_t)it * BK;
            // As[r][k]: 32 rows x 64 k = 2048; thread: k = tid & 63, r = (tid >> 6) + 4*i
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                int r = (tid >> 6) + 4 * i;
                int k = tid & 63;
                int64_t row = rbase + r;
                ra[i] = (row < c1 && k0 + k < d_in) ? __ldg(A + row * lda + acol0 + k) : 0.f;
            }
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                int idx = tid + i * NT;
                int r = idx >> 7, n = idx & 127;
                int64_t row = rbase + r;
                float v = 0.f;
                if (row < c1 && n0 + n < N) {
                    v = __ldg(dH + row * ldh + n0 + n);
                    if (relu && __ldg(H + row * ldh + n0 + n) <= 0.f) v = 0.f;
                }
                rb[i] = v;
            }
        };
        auto store = [&]() {
#pragma unroll
            for (int i = 0; i < 8; ++i) As[(tid >> 6) + 4 * i][tid & 63] = ra[i];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                int idx = tid + i * NT;
                Bs[idx >> 7][idx & 127] = rb[i];
            }
        };
        if (ntiles > 0) load(0);
        for (int it = 0; it < ntiles; ++it) {
            __syncthreads();
            store();
            __syncthreads();
            if (it + 1 < ntiles) load(it + 1);
            mma_tile(As, Bs, acc, tx, ty);
            if (do_db && ty == 0) {
#pragma unroll 4
                for (int k = 0; k < BK; ++k)
#pragma unroll
                    for (int j = 0; j < 8; ++j) cs[j] += Bs[k][out_col(tx, j)];
            }
        }
        float* Wp = dW + (int64_t)rg.slot_w[t][s] * wslot_stride;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            int k = k0 + ty * 4 + i;
            if (k >= d_in) continue;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                int n = n0 + out_col(tx, j);
                if (n < N) atomicAdd(Wp + (int64_t)k * ldw + n, acc[i][j]);
            }
        }
        if (do_db && ty == 0) {
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                int n = n0 + out_col(tx, j);
                if (n < N) atomicAdd(db + n, cs[j]);
            }
        }
        __syncthreads();
    }
}

}  // namespace gsb
