// sample.cu -- per-etype fanout sampling into message-flow blocks + relabel, all sizes
// device-resident (no host sync), sm_100a.  Contract: include/gsb.h "Mini-batch sampling".
//
// Per hop h (frontier D_h, type-grouped):
//   count   : thread per (dst j, slot s) -> c = min(f, deg'), marks map[gid(j)] = j
//   scan    : seg_ptr = exclusive_scan(c)                     (count's block totals + block scans)
//   fill    : warp per segment; Philox draws on lanes, Floyd resolved with shfl/ballot,
//             bitonic sort of the chosen ranks, coalesced writes; marks new sources in a
//             bitmap over the global id space
//   rank    : popcount prefix over the bitmap                 (block totals, then block scans)
//   meta    : per-type counts of new sources -> src row offsets (device HopMeta)
//   relabel : edge src gid -> src row (dst prefix via map, new via bitmap rank)
//   next    : writes D_{h+1} (dst prefix ++ ascending new) and clears map/bitmap
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "gsb_internal.cuh"
#include "rng.cuh"

namespace gsb {


enum { ERR_NONE = 0, ERR_GROUPING = 1, ERR_RANGE = 2, ERR_CAPACITY = 3, ERR_DUPLICATE = 4 };

// ------------------------------------------------------------------------------------
// LP exclusion set: sorted keys (flag << 62 | dst_gid << 31 | src_gid); flag 0 applies
// to segments of excl_etype, flag 1 to excl_rev_etype (R-excl).  Gids < 2^31.
// ------------------------------------------------------------------------------------
struct Excl {
    const uint64_t* keys;
    int64_t n;
    int32_t etype, rev;
    const int64_t* lo;    // [n] first excluded position of key k inside its dst segment
    const int64_t* cum;   // [n+1] exclusive prefix of the range lengths (duplicates: length 0)
};

// start of a sample: fold the previous sample's latch into the sticky word, clear the latch
__global__ void err_roll_kernel(int* __restrict__ err) {
    GSB_PDL_ENTRY();
    if (threadIdx.x == 0) {
        err[1] |= err[0];
        err[0] = 0;
    }
}

// Position range of every sorted exclusion key inside its destination's CSC segment
// (one binary search pair per key, once per batch).  Duplicate keys get an empty range at the
// previous key's end so that (lo - cum) stays non-decreasing within a segment.
__global__ void excl_ranges_kernel(GraphDev g, const uint64_t* __restrict__ keys, int64_t n, int32_t etype,
                                   int32_t rev, int64_t* __restrict__ lo_out, int64_t* __restrict__ len_out) {
    GSB_PDL_ENTRY();
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k <= n; k += (int64_t)gridDim.x * blockDim.x) {
        if (k == n) {
            len_out[k] = 0;
            continue;
        }
        const uint64_t key = keys[k];
        int64_t lo = 0, hi = 0;
        if (key != ~0ull) {
            const int r = (key >> 62) ? rev : etype;
            const int64_t v = (int64_t)((key >> 31) & 0x7FFFFFFFull);
            const int64_t u = (int64_t)(key & 0x7FFFFFFFull);
            const int t = type_of(g, v);
            const int64_t vl = v - g.node_off[t];
            const CscSeg cs = csc_seg(g, r, t, vl);
            const int64_t deg = cs.deg;
            const int32_t ul = (int32_t)(u - g.node_off[g.src_t[r]]);
            const int32_t* seg = cs.seg;
            int64_t l = 0, h = deg;
            while (l < h) { int64_t m = (l + h) >> 1; if (seg[m] < ul) l = m + 1; else h = m; }
            lo = l;
            h = deg;
            while (l < h) { int64_t m = (l + h) >> 1; if (seg[m] < ul + 1) l = m + 1; else h = m; }
            hi = l;
            if (k > 0 && keys[k - 1] == key) lo = hi;   // duplicate pair: empty range
        }
        lo_out[k] = lo;
        len_out[k] = hi - lo;
    }
}

__global__ void excl_keys_kernel(const int64_t* __restrict__ u, const int64_t* __restrict__ v, int64_t n, int rev,
                                 uint64_t* __restrict__ keys) {
    GSB_PDL_ENTRY();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        keys[i] = ((uint64_t)v[i] << 31) | (uint64_t)u[i];
        keys[n + i] = rev ? ((1ull << 62) | ((uint64_t)u[i] << 31) | (uint64_t)v[i]) : ~0ull;
    }
}

__device__ __forceinline__ int64_t lower_bound_u64(const uint64_t* a, int64_t n, uint64_t key) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t m = (lo + hi) >> 1;
        if (a[m] < key) lo = m + 1; else hi = m;
    }
    return lo;
}

__device__ __forceinline__ int64_t lower_bound_i32(const int32_t* a, int64_t n, int32_t key) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t m = (lo + hi) >> 1;
        if (a[m] < key) lo = m + 1; else hi = m;
    }
    return lo;
}

// Range [k0, k1) of exclusion keys for segment (v, r); empty when r is not excluded.
__device__ __forceinline__ void excl_range(const Excl& x, int r, int64_t v, int64_t& k0, int64_t& k1) {
    k0 = k1 = 0;
    if (x.n == 0 || (r != x.etype && r != x.rev)) return;
    uint64_t flag = (r == x.etype) ? 0ull : (1ull << 62);
    uint64_t base = flag | ((uint64_t)v << 31);
    k0 = lower_bound_u64(x.keys, x.n, base);
    k1 = lower_bound_u64(x.keys, x.n, base + (1ull << 31));
}

// Excluded positions of the segment whose keys are [k0, k1): their ranges are disjoint and
// ascending (keys sorted by src, segment sorted by src).
__device__ __forceinline__ int64_t excl_count(const Excl& x, int64_t k0, int64_t k1, const int32_t*, int64_t,
                                              int64_t) {
    return x.cum[k1] - x.cum[k0];
}

// Map rank q among non-excluded positions to a segment position: p = q + (lengths of the
// ranges starting at or before the q-th non-excluded position); binary search over
// nonexcl_before(k) = lo_k - (cum_k - cum_k0), which is non-decreasing in k.
__device__ __forceinline__ int64_t excl_map(const Excl& x, int64_t k0, int64_t k1, const int32_t*, int64_t, int64_t,
                                            int64_t q) {
    const int64_t c0 = x.cum[k0];
    int64_t l = k0, h = k1;   // first k with nonexcl_before(k) > q
    while (l < h) {
        const int64_t m = (l + h) >> 1;
        if (x.lo[m] - (x.cum[m] - c0) <= q) l = m + 1; else h = m;
    }
    return q + (x.cum[l] - c0);
}

// ------------------------------------------------------------------------------------
// hop-1 setup: copy seeds into the arena, per-type offsets, grouping / range checks
// ------------------------------------------------------------------------------------
__global__ void __launch_bounds__(1024) seed_meta_kernel(GraphDev g, const int64_t* __restrict__ seeds, int64_t n_cap,
                                                         const int64_t* __restrict__ n_dev,
                                                         int64_t* __restrict__ d1, HopMeta* __restrict__ m,
                                                         int* __restrict__ err) {
    GSB_PDL_ENTRY();
    __shared__ unsigned long long cnt[kMaxT];
    // the error latch roll-over (err_roll_kernel) folded in: one block, done before any check
    if (threadIdx.x == 0) {
        err[1] |= err[0];
        err[0] = 0;
    }
    __syncthreads();
    int64_t n = n_dev ? *n_dev : n_cap;
    if (n > n_cap) {
        if (threadIdx.x == 0) atomicExch(err, ERR_CAPACITY);
        n = n_cap;
    }
    if (threadIdx.x < kMaxT) cnt[threadIdx.x] = 0;
    __syncthreads();
    const int64_t N = g.node_off[g.T];
    const int lane = threadIdx.x & 31;
    for (int64_t base = 0; base < n; base += blockDim.x) {
        const int64_t i = base + threadIdx.x;
        int t = -1;
        if (i < n) {
            int64_t v = seeds[i];
            d1[i] = v;
            if (v < 0 || v >= N) {
                atomicExch(err, ERR_RANGE);
            } else {
                t = type_of(g, v);
                if (i > 0) {
                    int64_t p = seeds[i - 1];
                    if (p >= 0 && p < N && type_of(g, p) > t) atomicExch(err, ERR_GROUPING);
                }
            }
        }
        // warp-aggregated per-type counts (one shared atomic per warp and type)
        for (int tt = 0; tt < g.T; ++tt) {
            unsigned b = __ballot_sync(0xffffffffu, t == tt);
            if (lane == 0 && b) atomicAdd(&cnt[tt], (unsigned long long)__popc(b));
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const bool bad = *(volatile int*)err != 0;   // latched above: sample nothing
        m->n_dst = bad ? 0 : n;
        m->dst_off[0] = 0;
        for (int t = 0; t < kMaxT; ++t)
            m->dst_off[t + 1] = m->dst_off[t] + ((!bad && t < g.T) ? (int64_t)cnt[t] : 0);
    }
}

// Large seed sets (full-graph inference chunks of 10^5-10^6 nodes): the same copy, checks and
// per-type counts over the whole grid (block counts added into the zeroed dst_off[t + 1]),
// then one thread turns the counts into offsets.  One block of seed_meta_kernel walked a
// 262k-seed chunk in 0.28 ms.
__global__ void __launch_bounds__(256) seed_scan_kernel(GraphDev g, const int64_t* __restrict__ seeds, int64_t n_cap,
                                                        const int64_t* __restrict__ n_dev, int64_t* __restrict__ d1,
                                                        HopMeta* __restrict__ m, int* __restrict__ err) {
    GSB_PDL_ENTRY();
    __shared__ unsigned long long cnt[kMaxT];
    int64_t n = n_dev ? *n_dev : n_cap;
    if (n > n_cap) {
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicExch(err, ERR_CAPACITY);
        n = n_cap;
    }
    if (threadIdx.x < kMaxT) cnt[threadIdx.x] = 0;
    __syncthreads();
    const int64_t N = g.node_off[g.T];
    const int lane = threadIdx.x & 31;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n; base += stride) {
        const int64_t i = base + threadIdx.x;
        int t = -1;
        if (i < n) {
            const int64_t v = seeds[i];
            d1[i] = v;
            if (v < 0 || v >= N) {
                atomicExch(err, ERR_RANGE);
            } else {
                t = type_of(g, v);
                if (i > 0) {
                    const int64_t p = seeds[i - 1];
                    if (p >= 0 && p < N && type_of(g, p) > t) atomicExch(err, ERR_GROUPING);
                }
            }
        }
        for (int tt = 0; tt < g.T; ++tt) {
            const unsigned b = __ballot_sync(0xffffffffu, t == tt);
            if (lane == 0 && b) atomicAdd(&cnt[tt], (unsigned long long)__popc(b));
        }
    }
    __syncthreads();
    if (threadIdx.x < g.T && cnt[threadIdx.x])
        atomicAdd(reinterpret_cast<unsigned long long*>(&m->dst_off[threadIdx.x + 1]), cnt[threadIdx.x]);
}

__global__ void seed_fin_kernel(int T, int64_t n_cap, const int64_t* __restrict__ n_dev, HopMeta* __restrict__ m,
                                const int* __restrict__ err) {
    GSB_PDL_ENTRY();
    if (threadIdx.x != 0) return;
    int64_t n = n_dev ? *n_dev : n_cap;
    if (n > n_cap) n = n_cap;
    const bool bad = *(volatile const int*)err != 0;
    m->n_dst = bad ? 0 : n;
    m->dst_off[0] = 0;
    for (int t = 0; t < kMaxT; ++t) {
        const int64_t c = (!bad && t < T) ? m->dst_off[t + 1] : 0;
        m->dst_off[t + 1] = m->dst_off[t] + c;
    }
}

// ------------------------------------------------------------------------------------
// count: thread per (dst j, slot s), then seg_ptr = exclusive_scan(cnt) in one more launch.
// Count block b owns the contiguous chunk [b*chunk, (b+1)*chunk) of the nseg+1 entries (thread
// per entry, as many blocks as the latency-bound lookups want) and writes its total btot[b]; scan
// block b owns kScanPerBlock count chunks and adds the totals of the earlier ones (replaces CUB's
// init + look-back scan, two launches).
// ------------------------------------------------------------------------------------
constexpr int kCntThreads = 256, kCntPer = 8, kCntTile = kCntThreads * kCntPer, kCntMaxBlocks = kNumSMs * 16;
constexpr int kScanPerBlock = kCntPer;   // count chunks (multiples of kCntThreads entries) per scan block

__device__ __forceinline__ int64_t count_one(const GraphDev& g, int64_t i, int64_t n, int S,
                                             const int64_t* __restrict__ dst_gid, int fanout, const Excl& ex,
                                             int32_t* __restrict__ map, int* __restrict__ err,
                                             CscSeg* __restrict__ segc) {
    const int64_t j = i / S;
    const int s = (int)(i - j * S);
    if (j >= n) return 0;
    const int64_t v = dst_gid[j];
    const int t = type_of(g, v);
    if (s == 0 && map) {      // map == null: serving another rank's requests (no relabel here)
        int32_t old = atomicExch(map + v, (int32_t)j);
        if (old != -1) atomicExch(err, ERR_DUPLICATE);
    }
    if (s >= g.n_slots[t]) return 0;
    const int r = g.slot_etype[t][s];
    const int64_t vl = v - g.node_off[t];
    const CscSeg cs = csc_seg(g, r, t, vl);
    if (segc) segc[i] = cs;     // fill reads the resolved segment here (a remote one: no second NVLink trip)
    int64_t deg = cs.deg;
    int64_t k0, k1;
    excl_range(ex, r, v, k0, k1);
    if (k1 > k0) deg -= excl_count(ex, k0, k1, cs.seg, deg, g.node_off[g.src_t[r]]);
    return (fanout < 0 || deg <= fanout) ? deg : fanout;
}

// block-wide int64 sum over kCntThreads threads (valid in every thread)
__device__ __forceinline__ int64_t cnt_block_sum(int64_t v, int64_t* red) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    int64_t s = 0;
#pragma unroll
    for (int w = 0; w < kCntThreads / 32; ++w) s += red[w];
    __syncthreads();
    return s;
}

__global__ void __launch_bounds__(kCntThreads) count_kernel(GraphDev g, const HopMeta* __restrict__ m,
                                                            const int64_t* __restrict__ dst_gid, int64_t cap_dst,
                                                            int fanout, Excl ex, int32_t* __restrict__ map,
                                                            int64_t* __restrict__ cnt, int64_t chunk,
                                                            int64_t* __restrict__ btot, int* __restrict__ err,
                                                            CscSeg* __restrict__ segc) {
    GSB_PDL_ENTRY();
    __shared__ int64_t red[kCntThreads / 32];
    const int S = g.S;
    const int64_t n = (*(volatile int*)err) ? 0 : m->n_dst;
    const int64_t total = cap_dst * S;
    const int64_t i0 = blockIdx.x * chunk, i1 = min(i0 + chunk, total + 1);
    int64_t sum = 0;
    for (int64_t i = i0 + threadIdx.x; i < i1; i += kCntThreads) {
        const int64_t c = (i == total) ? 0 : count_one(g, i, n, S, dst_gid, fanout, ex, map, err, segc);
        cnt[i] = c;
        sum += c;
    }
    sum = cnt_block_sum(sum, red);
    if (threadIdx.x == 0) btot[blockIdx.x] = sum;
}

__global__ void __launch_bounds__(kCntThreads) count_scan_kernel(const int64_t* __restrict__ cnt, int64_t n_ent,
                                                                 int64_t chunk, const int64_t* __restrict__ btot,
                                                                 int nb_count, int64_t* __restrict__ seg_ptr) {
    GSB_PDL_ENTRY();
    __shared__ int64_t red[kCntThreads / 32];
    __shared__ int64_t wsum[kCntThreads / 32];
    int64_t off = 0;
    const int nprev = min((int)blockIdx.x * kScanPerBlock, nb_count);
    for (int b = threadIdx.x; b < nprev; b += kCntThreads) off += btot[b];
    off = cnt_block_sum(off, red);
    const int64_t i0 = blockIdx.x * chunk, i1 = min(i0 + chunk, n_ent);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int64_t t0 = i0; t0 < i1; t0 += kCntTile) {
        const int64_t base = t0 + (int64_t)threadIdx.x * kCntPer;
        int64_t c[kCntPer];
        if (base + kCntPer <= i1) {
            const longlong2* p = reinterpret_cast<const longlong2*>(cnt + base);
#pragma unroll
            for (int q = 0; q < kCntPer / 2; ++q) {
                const longlong2 x = p[q];
                c[2 * q] = x.x;
                c[2 * q + 1] = x.y;
            }
        } else {
#pragma unroll
            for (int k = 0; k < kCntPer; ++k) c[k] = (base + k < i1) ? cnt[base + k] : 0;
        }
        int64_t v = 0;
#pragma unroll
        for (int k = 0; k < kCntPer; ++k) v += c[k];
        int64_t inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) wsum[wid] = inc;
        __syncthreads();
        int64_t before = 0, tile = 0;
#pragma unroll
        for (int w = 0; w < kCntThreads / 32; ++w) {
            before += (w < wid) ? wsum[w] : 0;
            tile += wsum[w];
        }
        __syncthreads();
        int64_t r = off + before + inc - v;
        if (base + kCntPer <= i1) {
            longlong2* q = reinterpret_cast<longlong2*>(seg_ptr + base);
#pragma unroll
            for (int k = 0; k < kCntPer / 2; ++k) {
                const int64_t r0 = r, r1 = r0 + c[2 * k];
                r = r1 + c[2 * k + 1];
                q[k] = make_longlong2(r0, r1);
            }
        } else {
#pragma unroll
            for (int k = 0; k < kCntPer; ++k) {
                if (base + k < i1) seg_ptr[base + k] = r;
                r += c[k];
            }
        }
        off += tile;
    }
}

// ------------------------------------------------------------------------------------
// fill: one group of G lanes per segment (G >= fanout: 8, 16 or 32)
// ------------------------------------------------------------------------------------
#ifndef GSB_FILL_MINB
#define GSB_FILL_MINB 8      // 32 registers: 8 blocks / SM (46 registers at 5: sample_fill 42.4 -> 39.7 us in the step)
#endif
template <int G>
__global__ void __launch_bounds__(256, GSB_FILL_MINB) fill_kernel(GraphDev g, const HopMeta* __restrict__ m,
                                                   const int64_t* __restrict__ dst_gid, int64_t cap_dst,
                                                   const int64_t* __restrict__ seg_ptr, int fanout, Excl ex,
                                                   uint64_t seed, uint32_t step_host, const uint32_t* step_dev, int hop,
                                                   const int32_t* __restrict__ map, uint32_t* __restrict__ bitmap,
                                                   int64_t* __restrict__ e_src_gid, int64_t* __restrict__ e_eid,
                                                   const int* __restrict__ err, int64_t cap,
                                                   const int64_t* __restrict__ xoff, int xworld, int xrank,
                                                   const CscSeg* __restrict__ segc) {
    GSB_PDL_ENTRY();
    const int S = g.S;
    const int lane = threadIdx.x & 31;
    const int gl = lane & (G - 1);                       // lane inside the group
    const unsigned gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));
    const int64_t n = (*(volatile const int*)err) ? 0 : m->n_dst;
    const uint32_t step0 = step_dev ? *step_dev : step_host;
    const int64_t nseg = n * S;
    const int64_t groups = ((int64_t)gridDim.x * blockDim.x) / G;
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / G; i < nseg; i += groups) {
        const int64_t base = seg_ptr[i];
        const int64_t c = seg_ptr[i + 1] - base;
        if (c == 0) continue;
        const int64_t j = i / S;
        const int s = (int)(i - j * S);
        // serving requests (xoff): row j came from rank w, whose step word is this rank's
        // shifted by w - xrank (ranks step in lockstep, word = step * world + rank)
        uint32_t step = step0;
        if (xoff) {
            int w = 0;
            for (int k = 1; k < xworld; ++k) w += (j >= xoff[k]) ? 1 : 0;
            step = step0 + (uint32_t)(w - xrank);
        }
        const int64_t v = dst_gid[j];
        const int t = type_of(g, v);
        const int r = g.slot_etype[t][s];
        const int64_t vl = v - g.node_off[t];
        const CscSeg cs = segc ? segc[i] : csc_seg(g, r, t, vl);
        const int64_t deg = cs.deg;
        const int32_t* seg = cs.seg;
        const int64_t src_off = g.node_off[g.src_t[r]];
        int64_t k0, k1;
        excl_range(ex, r, v, k0, k1);
        const bool has_ex = k1 > k0;
        const int64_t degp = has_ex ? deg - excl_count(ex, k0, k1, seg, deg, src_off) : deg;
        if (c == degp) {
            // every non-excluded in-edge, ascending; beyond cap: fill_tail_kernel
            const int64_t ce = min(c, cap);
            for (int64_t q = gl; q < ce; q += G) {
                int64_t p = has_ex ? excl_map(ex, k0, k1, seg, deg, src_off, q) : q;
                int64_t u = src_off + seg[p];
                e_src_gid[base + q] = u;
                e_eid[base + q] = cs.eid0 + p;
                if (map && map[u] < 0) {
                    uint32_t bit = 1u << (u & 31);
                    if (!(bitmap[u >> 5] & bit)) atomicOr(bitmap + (u >> 5), bit);
                }
            }
            continue;
        }
        // Floyd (R-floyd): draw i (group lane i) is unif(j_i + 1), j_i = deg' - c + i
        const int cc = (int)c;  // c <= fanout <= G
        const int32_t jj = (int32_t)(degp - cc + gl);
        int32_t tdraw = 0;
        if (gl < cc) {
            uint32_t c2 = ((uint32_t)(r & 0xFFF) << 20) | ((uint32_t)(hop & 0xF) << 16) | (uint32_t)gl;
            uint64_t x = keyed_u64(seed, (uint32_t)(uint64_t)v, (uint32_t)((uint64_t)v >> 32), c2, step);
            tdraw = (int32_t)__umul64hi(x, (uint64_t)(jj + 1));
        }
        int32_t sel = INT32_MAX;
        for (int k = 0; k < cc; ++k) {
            int32_t tk = __shfl_sync(gmask, tdraw, k, G);
            unsigned hit = __ballot_sync(gmask, gl < k && sel == tk) & gmask;
            if (gl == k) sel = hit ? jj : tk;
        }
        // bitonic sort of sel across the group (ascending; unused lanes hold INT32_MAX)
#pragma unroll
        for (int kk = 2; kk <= G; kk <<= 1) {
#pragma unroll
            for (int jb = kk >> 1; jb > 0; jb >>= 1) {
                int32_t o = __shfl_xor_sync(gmask, sel, jb, G);
                bool up = (gl & kk) == 0 || kk == G;
                bool lower = (gl & jb) == 0;
                sel = (lower == up) ? min(sel, o) : max(sel, o);
            }
        }
        if (gl < cc) {
            int64_t p = has_ex ? excl_map(ex, k0, k1, seg, deg, src_off, sel) : sel;
            int64_t u = src_off + seg[p];
            e_src_gid[base + gl] = u;
            e_eid[base + gl] = cs.eid0 + p;
            if (map && map[u] < 0) {
                uint32_t bit = 1u << (u & 31);
                if (!(bitmap[u >> 5] & bit)) atomicOr(bitmap + (u >> 5), bit);
            }
        }
    }
}

// Fanout ALL (and fanouts above kFillCap) copy whole neighbourhoods; a power-law hub's
// segment (10^5 edges) would serialise one lane group.  fill_kernel copies the first kFillCap
// edges of each segment; here the hop's flat edge range is cut into pieces of kFillCap edges
// and a warp per piece copies the edges in it that lie beyond kFillCap of their segment.  A
// segment wholly inside a piece has <= kFillCap edges, so only the segments holding the
// piece's first and last edge qualify.  Segments longer than kFillCap are never Floyd draws
// (those hold c <= fanout <= 32 edges), so every such edge is the copy rule's.
constexpr int64_t kFillCap = 256;
#ifndef GSB_FILL_BPS
#define GSB_FILL_BPS 8
#endif

__global__ void __launch_bounds__(256) fill_tail_kernel(GraphDev g, const HopMeta* __restrict__ m,
                                                        const int64_t* __restrict__ dst_gid,
                                                        const int64_t* __restrict__ seg_ptr, Excl ex,
                                                        const int32_t* __restrict__ map, uint32_t* __restrict__ bitmap,
                                                        int64_t* __restrict__ e_src_gid, int64_t* __restrict__ e_eid,
                                                        const int* __restrict__ err) {
    GSB_PDL_ENTRY();
    const int S = g.S;
    const int lane = threadIdx.x & 31;
    const int64_t nseg = ((*(volatile const int*)err) ? 0 : m->n_dst) * S;
    const int64_t E = seg_ptr[nseg];
    const int64_t pieces = (E + kFillCap - 1) / kFillCap;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t k = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; k < pieces; k += warps) {
        const int64_t pa = k * kFillCap, pb = min(E, pa + kFillCap);
        const int64_t ia = seg_find(seg_ptr, 0, nseg, pa, lane);
        const int64_t ib = seg_find(seg_ptr, ia, nseg, pb - 1, lane);
        for (int64_t i = ia;; i = ib) {
            const int64_t base = seg_ptr[i];
            const int64_t q0 = max(pa, base + kFillCap) - base, q1 = min(pb, seg_ptr[i + 1]) - base;
            if (q0 < q1) {
                const int64_t j = i / S;
                const int s = (int)(i - j * S);
                const int64_t v = dst_gid[j];
                const int t = type_of(g, v);
                const int r = g.slot_etype[t][s];
                const int64_t vl = v - g.node_off[t];
                const CscSeg cs = csc_seg(g, r, t, vl);
                const int64_t deg = cs.deg;
                const int32_t* seg = cs.seg;
                const int64_t src_off = g.node_off[g.src_t[r]];
                int64_t k0, k1;
                excl_range(ex, r, v, k0, k1);
                const bool has_ex = k1 > k0;
                for (int64_t q = q0 + lane; q < q1; q += 32) {
                    const int64_t p = has_ex ? excl_map(ex, k0, k1, seg, deg, src_off, q) : q;
                    const int64_t u = src_off + seg[p];
                    e_src_gid[base + q] = u;
                    e_eid[base + q] = cs.eid0 + p;
                    if (map[u] < 0) {
                        const uint32_t bit = 1u << (u & 31);
                        if (!(bitmap[u >> 5] & bit)) atomicOr(bitmap + (u >> 5), bit);
                    }
                }
            }
            if (i == ib) break;
        }
    }
}

// ------------------------------------------------------------------------------------
// Transposed (by-source) CSR of a block (§8(a) a4): the backward scatter of a hidden layer
// then gathers, per source row, its edges' contributions in ascending edge order -- plain
// stores, no atomics, no memset, bit-reproducible (SPEC S:L281-284 by-src CSR).
// ------------------------------------------------------------------------------------
__global__ void tcsr_prep_kernel(const HopMeta* __restrict__ m, const int64_t* __restrict__ seg_ptr, int S,
                                 const int32_t* __restrict__ e_src, int64_t cap_edges, int32_t* __restrict__ e_seg,
                                 int32_t* __restrict__ key, int32_t* __restrict__ val) {
    GSB_PDL_ENTRY();
    const int64_t E = m->n_edges, nseg = m->n_dst * S;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < cap_edges; e += stride) {
        key[e] = e < E ? e_src[e] : INT32_MAX;
        val[e] = (int32_t)e;
    }
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nseg; i += stride)
        for (int64_t e = seg_ptr[i]; e < seg_ptr[i + 1]; ++e) e_seg[e] = (int32_t)i;
}

// t_ptr over the sorted keys; per transposed position k the edge's segment id (t_seg, in the
// freed key buffer) and 1 / its segment count (t_inv, in the freed value buffer), so the
// scatter's only dependent load is the gradient row
__global__ void tcsr_ptr_kernel(const HopMeta* __restrict__ m, const int32_t* __restrict__ key, int64_t cap_src,
                                int32_t* __restrict__ t_ptr, const int32_t* __restrict__ t_edge,
                                const int32_t* __restrict__ e_seg, const int64_t* __restrict__ seg_ptr,
                                int32_t* __restrict__ t_seg, int32_t* __restrict__ t_inv) {
    GSB_PDL_ENTRY();
    const int64_t E = m->n_edges;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u <= cap_src; u += stride) {
        int64_t lo = 0, hi = E;
        while (lo < hi) {
            const int64_t mid = (lo + hi) >> 1;
            if (key[mid] < u) lo = mid + 1; else hi = mid;
        }
        t_ptr[u] = (int32_t)lo;
    }
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < E; k += stride) {
        const int32_t i = e_seg[t_edge[k]];
        t_seg[k] = i;
        t_inv[k] = __float_as_int(1.f / (float)(seg_ptr[i + 1] - seg_ptr[i]));
    }
}

// ------------------------------------------------------------------------------------
// NCCL frontier exchange (§8(e) C2/C3, gsb_blocks_set_exchange): requester side buckets the
// hop's frontier by owner (K11); the owner runs count / scan / fill on the requests it
// received (keyed draws with the requester's step word: the same blocks as a whole-graph
// sampler); the requester unpacks the returned counts and edges into frontier order.
// ------------------------------------------------------------------------------------
__device__ __forceinline__ int x_owner(const GraphDev& g, int64_t v) {
    const CscPeers& P = *g.cpeers;
    const int t = type_of(g, v);
    const int64_t vl = v - g.node_off[t];
    int w = 0;
    for (int k = 1; k < P.world; ++k) w += (vl >= P.lo[t][k]) ? 1 : 0;
    return w;
}

// per-owner request counts, one shared atomic per (warp, owner)
__global__ void x_owner_count_kernel(GraphDev g, const HopMeta* __restrict__ m, const int64_t* __restrict__ dst_gid,
                                     int world, unsigned long long* __restrict__ cnt) {
    GSB_PDL_ENTRY();
    __shared__ unsigned long long sc[kMaxPeers];
    if (threadIdx.x < kMaxPeers) sc[threadIdx.x] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t n = m->n_dst;
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x; b < n; b += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = b + threadIdx.x;
        const int w = i < n ? x_owner(g, dst_gid[i]) : -1;
        for (int o = 0; o < world; ++o) {
            const unsigned bal = __ballot_sync(0xffffffffu, w == o);
            if (lane == 0 && bal) atomicAdd(&sc[o], (unsigned long long)__popc(bal));
        }
    }
    __syncthreads();
    if (threadIdx.x < world && sc[threadIdx.x]) atomicAdd(&cnt[threadIdx.x], sc[threadIdx.x]);
}

__global__ void x_scatter_kernel(GraphDev g, const HopMeta* __restrict__ m, const int64_t* __restrict__ dst_gid,
                                 int world, const unsigned long long* __restrict__ cnt,
                                 unsigned long long* __restrict__ cursor, int64_t* __restrict__ req_send,
                                 int32_t* __restrict__ perm) {
    GSB_PDL_ENTRY();
    __shared__ unsigned long long base[kMaxPeers];
    if (threadIdx.x == 0) {
        unsigned long long a = 0;
        for (int w = 0; w < world; ++w) {
            base[w] = a;
            a += cnt[w];
        }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const int64_t n = m->n_dst;
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x; b < n; b += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = b + threadIdx.x;
        int64_t v = 0;
        int w = -1;
        if (i < n) {
            v = dst_gid[i];
            w = x_owner(g, v);
        }
        for (int o = 0; o < world; ++o) {
            const unsigned bal = __ballot_sync(0xffffffffu, w == o);
            if (!bal) continue;
            const int leader = __ffs(bal) - 1;
            unsigned long long start = 0;
            if (lane == leader) start = atomicAdd(&cursor[o], (unsigned long long)__popc(bal));
            start = __shfl_sync(0xffffffffu, start, leader);
            if (w == o) {
                const int64_t pos = (int64_t)(base[o] + start + __popc(bal & lt));
                req_send[pos] = v;
                perm[i] = (int32_t)pos;
            }
        }
    }
}

// edges to return to each requesting rank: its requests are rows [xoff[w], xoff[w+1])
__global__ void x_wcnt_kernel(const int64_t* __restrict__ srv_seg, const int64_t* __restrict__ xoff, int world, int S,
                              int64_t* __restrict__ wcnt) {
    GSB_PDL_ENTRY();
    const int w = threadIdx.x;
    if (w < world) wcnt[w] = srv_seg[xoff[w + 1] * S] - srv_seg[xoff[w] * S];
}

// requester: per (frontier row, slot) counts from the owners' replies; dst map for relabel;
// entries past the live rows are zero (the scan runs over the capacity)
__global__ void x_unpack_count_kernel(const HopMeta* __restrict__ m, const int64_t* __restrict__ dst_gid,
                                      const int32_t* __restrict__ perm, const int64_t* __restrict__ resp_cnt, int S,
                                      int64_t cap_entries, int32_t* __restrict__ map, int64_t* __restrict__ cnt,
                                      int* __restrict__ err) {
    GSB_PDL_ENTRY();
    const int64_t n = (*(volatile const int*)err) ? 0 : m->n_dst;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= cap_entries;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = i / S;
        const int s = (int)(i - j * S);
        if (j >= n) {
            cnt[i] = 0;
            continue;
        }
        cnt[i] = resp_cnt[(int64_t)perm[j] * S + s];
        if (s == 0) {
            const int32_t old = atomicExch(map + dst_gid[j], (int32_t)j);
            if (old != -1) atomicExch(err, ERR_DUPLICATE);
        }
    }
}

// requester: copy every segment's returned edges into frontier order, mark new sources
__global__ void x_unpack_fill_kernel(const HopMeta* __restrict__ m, const int32_t* __restrict__ perm, int S,
                                     const int64_t* __restrict__ seg_ptr, const int64_t* __restrict__ resp_seg,
                                     const int64_t* __restrict__ resp_gid, const int64_t* __restrict__ resp_eid,
                                     const int32_t* __restrict__ map, uint32_t* __restrict__ bitmap,
                                     int64_t* __restrict__ e_src_gid, int64_t* __restrict__ e_eid,
                                     const int* __restrict__ err) {
    GSB_PDL_ENTRY();
    const int64_t n = (*(volatile const int*)err) ? 0 : m->n_dst;
    const int64_t nseg = n * S;
    const int lane = threadIdx.x & 31;
    const int64_t warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < nseg; i += warps) {
        const int64_t d0 = seg_ptr[i], c = seg_ptr[i + 1] - d0;
        if (c == 0) continue;
        const int64_t j = i / S;
        const int s = (int)(i - j * S);
        const int64_t r0 = resp_seg[(int64_t)perm[j] * S + s];
        for (int64_t q = lane; q < c; q += 32) {
            const int64_t u = resp_gid[r0 + q];
            e_src_gid[d0 + q] = u;
            e_eid[d0 + q] = resp_eid[r0 + q];
            if (map[u] < 0) {
                const uint32_t bit = 1u << (u & 31);
                if (!(bitmap[u >> 5] & bit)) atomicOr(bitmap + (u >> 5), bit);
            }
        }
    }
}

// ------------------------------------------------------------------------------------
// rank / meta / relabel / next frontier
// ------------------------------------------------------------------------------------
// Word ranks of the visited bitmap in two launches (replaces popc + CUB's init + scan, three
// launches): wrank[w] = sum_{v < w} popc(bitmap[v]) for w in [0, n_words], words >= n_words
// count 0.  Block b owns the words [b*chunk, (b+1)*chunk) (chunk = whole tiles of
// kRankTile words, kRankPerThread consecutive words per thread, at most kRankMaxBlocks
// blocks); rank_sum_kernel writes the block's popcount total btot[b], rank_scan_kernel adds
// the totals of the earlier blocks.
constexpr int kRankThreads = 256, kRankPerThread = 4, kRankTile = kRankThreads * kRankPerThread;
constexpr int kRankMaxBlocks = kNumSMs * 4;

__device__ __forceinline__ void rank_load(const uint32_t* __restrict__ bitmap, int64_t n_words, int64_t base,
                                          uint32_t (&c)[kRankPerThread]) {
    if (base + kRankPerThread <= n_words) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(bitmap + base));
        c[0] = __popc(v.x); c[1] = __popc(v.y); c[2] = __popc(v.z); c[3] = __popc(v.w);
    } else {
#pragma unroll
        for (int i = 0; i < kRankPerThread; ++i) c[i] = (base + i < n_words) ? __popc(bitmap[base + i]) : 0;
    }
}

// block-wide sum over kRankThreads threads (result valid in every thread)
__device__ __forceinline__ int rank_block_sum(int v, int* red) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    int s = 0;
#pragma unroll
    for (int w = 0; w < kRankThreads / 32; ++w) s += red[w];
    __syncthreads();
    return s;
}

__global__ void __launch_bounds__(kRankThreads) rank_sum_kernel(const uint32_t* __restrict__ bitmap, int64_t n_words,
                                                                int64_t chunk, int32_t* __restrict__ btot) {
    GSB_PDL_ENTRY();
    __shared__ int red[kRankThreads / 32];
    const int64_t w0 = blockIdx.x * chunk, w1 = min(w0 + chunk, n_words + 1);
    int v = 0;
    for (int64_t base = w0 + (int64_t)threadIdx.x * kRankPerThread; base < w1; base += kRankTile) {
        uint32_t c[kRankPerThread];
        rank_load(bitmap, n_words, base, c);
#pragma unroll
        for (int i = 0; i < kRankPerThread; ++i) v += (int)c[i];
    }
    v = rank_block_sum(v, red);
    if (threadIdx.x == 0) btot[blockIdx.x] = v;
}

__global__ void __launch_bounds__(kRankThreads) rank_scan_kernel(const uint32_t* __restrict__ bitmap, int64_t n_words,
                                                                 int64_t chunk, const int32_t* __restrict__ btot,
                                                                 int32_t* __restrict__ wrank) {
    GSB_PDL_ENTRY();
    __shared__ int red[kRankThreads / 32];
    __shared__ int wsum[kRankThreads / 32];
    int off = 0;   // words of earlier blocks
    for (int b = threadIdx.x; b < (int)blockIdx.x; b += kRankThreads) off += btot[b];
    off = rank_block_sum(off, red);
    const int64_t w0 = blockIdx.x * chunk, w1 = min(w0 + chunk, n_words + 1);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int64_t t0 = w0; t0 < w1; t0 += kRankTile) {
        const int64_t base = t0 + (int64_t)threadIdx.x * kRankPerThread;
        uint32_t c[kRankPerThread];
        rank_load(bitmap, n_words, base, c);
        const int v = (int)(c[0] + c[1] + c[2] + c[3]);
        // exclusive scan of v over the block: warp inclusive scan, then warp totals
        int inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) wsum[wid] = inc;
        __syncthreads();
        int before = 0, tile = 0;
#pragma unroll
        for (int w = 0; w < kRankThreads / 32; ++w) {
            before += (w < wid) ? wsum[w] : 0;
            tile += wsum[w];
        }
        __syncthreads();
        int r0 = off + before + inc - v;
        const int r1 = r0 + (int)c[0], r2 = r1 + (int)c[1], r3 = r2 + (int)c[2];
        if (base + kRankPerThread <= w1) {
            *reinterpret_cast<int4*>(wrank + base) = make_int4(r0, r1, r2, r3);
        } else {
            const int r[4] = {r0, r1, r2, r3};
#pragma unroll
            for (int i = 0; i < kRankPerThread; ++i)
                if (base + i < w1) wrank[base + i] = r[i];
        }
        off += tile;
    }
}

__device__ __forceinline__ int64_t bit_rank(const uint32_t* bitmap, const int32_t* wrank, int64_t x) {
    int64_t w = x >> 5;
    int b = (int)(x & 31);
    int64_t r = wrank[w];
    if (b) r += __popc(bitmap[w] & ((1u << b) - 1u));
    return r;
}

// hop metadata from the finished word ranks, run by one warp (threads 0..31 of a block)
__device__ __forceinline__ void hop_meta_body(const GraphDev& g, HopMeta* __restrict__ m, HopMeta* __restrict__ next,
                                              const int64_t* __restrict__ seg_ptr, int64_t nseg_cap,
                                              const uint32_t* __restrict__ bitmap, const int32_t* __restrict__ wrank,
                                              int64_t cap_src, int* __restrict__ err, int64_t* nn_s) {
    const int t = threadIdx.x;
    const bool bad = *(volatile int*)err != 0;
    if (!bad && t < kMaxT) {   // one thread per node type: new-source count via bitmap ranks
        int64_t nn = 0;
        if (t < g.T) {
            const int64_t lo = bit_rank(bitmap, wrank, g.node_off[t]);
            const int64_t hi = bit_rank(bitmap, wrank, g.node_off[t + 1]);
            m->new_base[t] = lo;
            nn = hi - lo;
        }
        nn_s[t] = nn;
    }
    __syncwarp();
    if (t != 0) return;
    if (bad) {   // latched: empty block and frontier (kernels downstream see 0 rows)
        m->n_edges = 0;
        m->n_src = 0;
        for (int k = 0; k <= kMaxT; ++k) m->src_off[k] = 0;
        if (next) {
            next->n_dst = 0;
            for (int k = 0; k <= kMaxT; ++k) next->dst_off[k] = 0;
        }
        return;
    }
    m->n_edges = seg_ptr[nseg_cap];
    int64_t off = 0;
    m->src_off[0] = 0;
    for (int k = 0; k < kMaxT; ++k) {
        off += (m->dst_off[k + 1] - m->dst_off[k]) + nn_s[k];
        m->src_off[k + 1] = off;
    }
    m->n_src = off;
    if (m->n_src > cap_src) {
        atomicExch(err, ERR_CAPACITY);
        m->n_src = cap_src;
    }
    if (next) {
        next->n_dst = m->n_src;
        for (int k = 0; k <= kMaxT; ++k) next->dst_off[k] = m->src_off[k];
    }
}

__global__ void hop_meta_kernel(GraphDev g, HopMeta* __restrict__ m, HopMeta* __restrict__ next,
                                const int64_t* __restrict__ seg_ptr, int64_t nseg_cap, const uint32_t* __restrict__ bitmap,
                                const int32_t* __restrict__ wrank, int64_t cap_src, int* __restrict__ err) {
    GSB_PDL_ENTRY();
    __shared__ int64_t nn_s[kMaxT];
    if (threadIdx.x < 32) hop_meta_body(g, m, next, seg_ptr, nseg_cap, bitmap, wrank, cap_src, err, nn_s);
}

// One launch for the word ranks and the hop metadata (rank_sum + rank_scan + hop_meta): every
// block sums its chunk's bit counts, publishes the total in an epoch-tagged flag, adds the
// totals of the blocks before it (decoupled look-back; blocks are scheduled in index order, so
// a block only waits on blocks already resident or done), writes its words' exclusive ranks, and
// the last block to finish (ticket) builds the hop metadata and advances the epoch.
__global__ void __launch_bounds__(kRankThreads) rank_fused_kernel(
    GraphDev g, const uint32_t* __restrict__ bitmap, int64_t n_words, int64_t chunk, int32_t* __restrict__ wrank,
    unsigned long long* __restrict__ flags, HopMeta* __restrict__ m, HopMeta* __restrict__ next,
    const int64_t* __restrict__ seg_ptr, int64_t nseg_cap, int64_t cap_src, int* __restrict__ err) {
    GSB_PDL_ENTRY();
    __shared__ int red[kRankThreads / 32];
    __shared__ int wsum[kRankThreads / 32];
    __shared__ int64_t nn_s[kMaxT];
    __shared__ unsigned last;
    unsigned* epoch_p = reinterpret_cast<unsigned*>(flags + kRankMaxBlocks);
    unsigned* ticket_p = epoch_p + 1;
    const unsigned long long tag = (unsigned long long)(*(volatile unsigned*)epoch_p + 1u) << 32;
    const int64_t w0 = blockIdx.x * chunk, w1 = min(w0 + chunk, n_words + 1);
    // (1) this block's total, published
    int v = 0;
    for (int64_t base = w0 + (int64_t)threadIdx.x * kRankPerThread; base < w1; base += kRankTile) {
        uint32_t c[kRankPerThread];
        rank_load(bitmap, n_words, base, c);
#pragma unroll
        for (int i = 0; i < kRankPerThread; ++i) v += (int)c[i];
    }
    v = rank_block_sum(v, red);
    if (threadIdx.x == 0) {
        __threadfence();
        atomicExch(flags + blockIdx.x, tag | (unsigned)v);
    }
    // (2) totals of the earlier blocks
    int off = 0;
    for (int b = threadIdx.x; b < (int)blockIdx.x; b += kRankThreads) {
        unsigned long long f;
        do {
            f = *(volatile unsigned long long*)(flags + b);
        } while ((f & 0xFFFFFFFF00000000ull) != tag);
        off += (int)(unsigned)f;
    }
    off = rank_block_sum(off, red);
    // (3) exclusive word ranks of the chunk
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int64_t t0 = w0; t0 < w1; t0 += kRankTile) {
        const int64_t base = t0 + (int64_t)threadIdx.x * kRankPerThread;
        uint32_t c[kRankPerThread];
        rank_load(bitmap, n_words, base, c);
        const int vv = (int)(c[0] + c[1] + c[2] + c[3]);
        int inc = vv;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        if (lane == 31) wsum[wid] = inc;
        __syncthreads();
        int before = 0, tile = 0;
#pragma unroll
        for (int w = 0; w < kRankThreads / 32; ++w) {
            before += (w < wid) ? wsum[w] : 0;
            tile += wsum[w];
        }
        __syncthreads();
        const int r0 = off + before + inc - vv;
        const int r1 = r0 + (int)c[0], r2 = r1 + (int)c[1], r3 = r2 + (int)c[2];
        if (base + kRankPerThread <= w1) {
            *reinterpret_cast<int4*>(wrank + base) = make_int4(r0, r1, r2, r3);
        } else {
            const int r[4] = {r0, r1, r2, r3};
#pragma unroll
            for (int i = 0; i < kRankPerThread; ++i)
                if (base + i < w1) wrank[base + i] = r[i];
        }
        off += tile;
    }
    // (4) the last block: hop metadata, next epoch
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = (atomicAdd(ticket_p, 1u) == gridDim.x - 1) ? 1u : 0u;
    __syncthreads();
    if (!last) return;
    __threadfence();
    if (threadIdx.x < 32) hop_meta_body(g, m, next, seg_ptr, nseg_cap, bitmap, wrank, cap_src, err, nn_s);
    if (threadIdx.x == 0) {
        *ticket_p = 0;
        *epoch_p = *epoch_p + 1u;
    }
}

__global__ void __launch_bounds__(256) relabel_kernel(GraphDev g, const HopMeta* __restrict__ m,
                                                      const int64_t* __restrict__ e_src_gid,
                                                      const int32_t* __restrict__ map,
                                                      const uint32_t* __restrict__ bitmap,
                                                      const int32_t* __restrict__ wrank, int32_t* __restrict__ e_src) {
    GSB_PDL_ENTRY();
    const int64_t E = m->n_edges;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < E; e += (int64_t)gridDim.x * blockDim.x) {
        int64_t u = e_src_gid[e];
        int t = type_of(g, u);
        int32_t mj = map[u];
        int64_t row;
        if (mj >= 0)
            row = m->src_off[t] + (mj - m->dst_off[t]);
        else
            row = m->src_off[t] + (m->dst_off[t + 1] - m->dst_off[t]) + (bit_rank(bitmap, wrank, u) - m->new_base[t]);
        e_src[e] = (int32_t)row;
    }
}

__global__ void __launch_bounds__(256) next_frontier_kernel(GraphDev g, const HopMeta* __restrict__ m,
                                                            const int64_t* __restrict__ dst_gid,
                                                            int32_t* __restrict__ map, uint32_t* __restrict__ bitmap,
                                                            const int32_t* __restrict__ wrank, int64_t n_words,
                                                            int64_t cap_src, int64_t* __restrict__ src_gid) {
    GSB_PDL_ENTRY();
    const int64_t n = m->n_dst;
    const int64_t work = n > n_words ? n : n_words;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < work; i += (int64_t)gridDim.x * blockDim.x) {
        if (i < n) {
            int64_t v = dst_gid[i];
            int t = type_of(g, v);
            int64_t row = m->src_off[t] + (i - m->dst_off[t]);
            if (row < cap_src) src_gid[row] = v;
            map[v] = -1;
        }
        if (i < n_words) {
            uint32_t bits = bitmap[i];
            if (bits) {
                int64_t k = wrank[i];
                while (bits) {
                    int b = __ffs(bits) - 1;
                    bits &= bits - 1;
                    int64_t u = i * 32 + b;
                    int t = type_of(g, u);
                    int64_t row = m->src_off[t] + (m->dst_off[t + 1] - m->dst_off[t]) + (k - m->new_base[t]);
                    if (row < cap_src) src_gid[row] = u;
                    ++k;
                }
                bitmap[i] = 0;
            }
        }
    }
}

__global__ void init_arena_kernel(int32_t* __restrict__ map, int64_t n, uint32_t* __restrict__ bitmap, int64_t n_words,
                                  int* __restrict__ err) {
    GSB_PDL_ENTRY();
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n || i < n_words;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (i < n) map[i] = -1;
        if (i < n_words) bitmap[i] = 0;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) err[0] = err[1] = 0;
}

// the fused rank kernel's int64 block flags (+ epoch, ticket), 8-B aligned after the ranks
static int64_t* rank_flags(const Blocks* B, void* arena) {
    const uintptr_t p = reinterpret_cast<uintptr_t>(at<int32_t>(arena, B->off_wrank) + B->n_words + 1 + kRankMaxBlocks);
    return reinterpret_cast<int64_t*>((p + 7) & ~uintptr_t(7));
}

HopBufs Blocks::hop(int h, void* arena) const {
    HopBufs b;
    b.cap_dst = cap_dst[h];
    b.cap_seeds = cap_dst[1];
    b.cap_edges = cap_edges[h];
    b.cap_src = cap_dst[h + 1];
    b.meta = at<HopMeta>(arena, off_meta[h]);
    b.dst_gid = (h == 1) ? at<int64_t>(arena, off_seed) : at<int64_t>(arena, off_src[h - 1]);
    b.cnt = at<int64_t>(arena, off_cnt[h]);
    b.seg_ptr = at<int64_t>(arena, off_seg[h]);
    b.e_src_gid = at<int64_t>(arena, off_esrcgid[h]);
    b.e_eid = at<int64_t>(arena, off_eeid[h]);
    b.e_src = at<int32_t>(arena, off_esrc[h]);
    b.src_gid = at<int64_t>(arena, off_src[h]);
    b.segc = at<CscSeg>(arena, off_segc[h]);
    if (off_tcsr[h]) {
        int32_t* t = at<int32_t>(arena, off_tcsr[h]);
        b.e_seg = t;
        b.t_key = t + cap_edges[h];
        b.t_key2 = t + 2 * cap_edges[h];
        b.t_val = t + 3 * cap_edges[h];
        b.t_edge = t + 4 * cap_edges[h];
        b.t_ptr = t + 5 * cap_edges[h];
    } else {
        b.e_seg = b.t_key = b.t_key2 = b.t_val = b.t_edge = b.t_ptr = nullptr;
    }
    return b;
}

// One hop of the NCCL exchange mode (see the kernels above): bucket -> callback phase 0
// (request all-to-all) -> owner-side count / scan / fill of the received requests -> callback
// phase 1 (reply all-to-alls) -> unpack into this rank's hop buffers.  Host-synchronous at
// the two callbacks (the exchange sizes are read on the host); not CUDA-graph capturable.
static gsb_status exchange_hop(Blocks* B, const gsb_sample_args* a, const HopBufs& hb, int h, int f, int S,
                               uint64_t rng_seed, int32_t* map, uint32_t* bitmap, int* err, void* cub_tmp,
                               cudaStream_t s) {
    const GraphDev& g = B->g->dev;
    Xchg& x = B->x;
    GSB_CHECK_ARG(f >= 1 && f <= GSB_MAX_FANOUT, "exchange mode needs a fanout in [1, %d]", GSB_MAX_FANOUT);
    GSB_CHECK_ARG(g.cpeers, "exchange mode needs the partition bounds (gsb_graph_set_csc_peers)");
    const Excl ex0{nullptr, 0, -1, -2, nullptr, nullptr};
    // (1) bucket the frontier by owner
    GSB_CUDA(cudaMemsetAsync(x.send_cnt, 0, sizeof(int64_t) * x.world, s));
    GSB_CUDA(cudaMemsetAsync(x.cursor, 0, sizeof(int64_t) * x.world, s));
    const int gb = grid_for(hb.cap_dst, 256, kNumSMs * 4);
    GSB_LAUNCH("x_bucket", x_owner_count_kernel, gb, 256, 0, s, g, hb.meta, hb.dst_gid, x.world,
               reinterpret_cast<unsigned long long*>(x.send_cnt));
    GSB_LAUNCH("x_scatter", x_scatter_kernel, gb, 256, 0, s, g, hb.meta, hb.dst_gid, x.world,
               reinterpret_cast<const unsigned long long*>(x.send_cnt), reinterpret_cast<unsigned long long*>(x.cursor),
               x.req_send, x.req_perm);
    // (2) C2: requests to their owners
    int64_t cnt[kMaxPeers + 1] = {0};
    if (x.fn(x.user, 0, h, (void*)s, cnt) != 0) {
        set_error("exchange callback failed (phase 0, hop %d)", h);
        return GSB_ECALLBACK;
    }
    int64_t off[kMaxPeers + 1];
    off[0] = 0;
    for (int w = 0; w < x.world; ++w) off[w + 1] = off[w] + cnt[w];
    const int64_t n_recv = off[x.world];
    GSB_CHECK_ARG(n_recv <= x.cap_recv, "received %lld requests > capacity %lld", (long long)n_recv,
                  (long long)x.cap_recv);
    HopMeta hm;
    memset(&hm, 0, sizeof(hm));
    hm.n_dst = n_recv;
    GSB_CUDA(cudaMemcpyAsync(x.srv_meta, &hm, sizeof(HopMeta), cudaMemcpyHostToDevice, s));
    GSB_CUDA(cudaMemcpyAsync(x.xoff, off, sizeof(int64_t) * (x.world + 1), cudaMemcpyHostToDevice, s));
    // (3) serve: count / scan / fill over the received requests (no relabel state touched)
    const int64_t sseg = n_recv * S;
    {
        const int64_t chunk = ceil_div(ceil_div(sseg + 1, kCntThreads), kCntMaxBlocks) * kCntThreads;
        const int nb = (int)ceil_div(sseg + 1, chunk);
        const int nbs = (int)ceil_div(sseg + 1, chunk * kScanPerBlock);
        int64_t* btot = x.srv_cnt + sseg + 1;
        GSB_LAUNCH("x_serve_count", count_kernel, nb, kCntThreads, 0, s, g, x.srv_meta, x.req_recv, n_recv, f, ex0,
                   (int32_t*)nullptr, x.srv_cnt, chunk, btot, err, (CscSeg*)nullptr);
        GSB_LAUNCH("x_serve_scan", count_scan_kernel, nbs, kCntThreads, 0, s, x.srv_cnt, sseg + 1,
                   chunk * kScanPerBlock, btot, nb, x.srv_seg);
        const int G = f <= 8 ? 8 : (f <= 16 ? 16 : 32);
        const int grid = grid_for(std::max<int64_t>(sseg, 1) * G, 256, kNumSMs * GSB_FILL_BPS);
#define GSB_XFILL(GG)                                                                                            \
    GSB_LAUNCH("x_serve_fill", fill_kernel<GG>, grid, 256, 0, s, g, x.srv_meta, x.req_recv, n_recv, x.srv_seg, f,   \
               ex0, rng_seed, a->step, a->step_dev, h, (const int32_t*)nullptr, (uint32_t*)nullptr, x.srv_gid,     \
               x.srv_eid, err, INT64_MAX, (const int64_t*)x.xoff, x.world, x.rank, (const CscSeg*)nullptr)
        if (G == 8) GSB_XFILL(8);
        else if (G == 16) GSB_XFILL(16);
        else GSB_XFILL(32);
#undef GSB_XFILL
        GSB_LAUNCH("x_wcnt", x_wcnt_kernel, 1, 32, 0, s, x.srv_seg, x.xoff, x.world, S, x.srv_wcnt);
    }
    // (4) C3: replies back to the requesters
    GSB_CUDA(cudaMemsetAsync(x.resp_cnt, 0, sizeof(int64_t) * (size_t)(hb.cap_dst * S + 1), s));
    if (x.fn(x.user, 1, h, (void*)s, cnt) != 0) {
        set_error("exchange callback failed (phase 1, hop %d)", h);
        return GSB_ECALLBACK;
    }
    // (5) unpack into frontier order: counts -> seg_ptr; reply offsets; edges
    const int64_t nseg = hb.cap_dst * S;
    GSB_LAUNCH("x_unpack_count", x_unpack_count_kernel, grid_for(nseg + 1, 256, kNumSMs * 8), 256, 0, s, hb.meta,
               hb.dst_gid, x.req_perm, x.resp_cnt, S, nseg, map, hb.cnt, err);
    size_t cb = B->cub_bytes;
    GSB_CUDA(cub::DeviceScan::ExclusiveSum(cub_tmp, cb, hb.cnt, hb.seg_ptr, (int64_t)(nseg + 1), s));
    cb = B->cub_bytes;
    GSB_CUDA(cub::DeviceScan::ExclusiveSum(cub_tmp, cb, x.resp_cnt, x.resp_seg, (int64_t)(nseg + 1), s));
    count_launch(4);
    GSB_LAUNCH("x_unpack_fill", x_unpack_fill_kernel, grid_for(nseg * 32, 256, kNumSMs * 8), 256, 0, s, hb.meta,
               x.req_perm, S, hb.seg_ptr, x.resp_seg, x.resp_gid, x.resp_eid, map, bitmap, hb.e_src_gid, hb.e_eid,
               err);
    return GSB_OK;
}

}  // namespace gsb

using namespace gsb;

extern "C" {

gsb_status gsb_blocks_create(gsb_graph_t gh, int32_t L, const int32_t* fanouts, int64_t max_seeds, int64_t max_excl,
                             gsb_blocks_t* out) {
    Graph* G = reinterpret_cast<Graph*>(gh);
    GSB_CHECK_ARG(G && fanouts && out, "null argument");
    GSB_CHECK_ARG(L >= 1 && L <= kMaxL, "num_layers %d out of [1, %d]", L, kMaxL);
    GSB_CHECK_ARG(max_seeds >= 1 && max_excl >= 0, "bad capacities");
    GSB_CHECK_ARG(G->total_nodes < ((int64_t)1 << 31), "total node count must be < 2^31");
    for (int l = 0; l < L; ++l)
        GSB_CHECK_ARG(fanouts[l] == -1 || (fanouts[l] >= 1 && fanouts[l] <= GSB_MAX_FANOUT),
                      "fanout %d must be -1 or in [1, %d]", fanouts[l], GSB_MAX_FANOUT);
    for (int r = 0; r < G->dev.R; ++r)
        GSB_CHECK_ARG(G->dev.indptr[r] != nullptr, "CSC of etype %d not registered", r);
    Blocks* B = new Blocks();
    memset(B, 0, sizeof(Blocks));
    B->g = G;
    B->L = L;
    for (int l = 0; l < L; ++l) B->fanout[l] = fanouts[l];
    B->max_seeds = max_seeds;
    B->max_excl = max_excl;
    const int S = G->dev.S > 0 ? G->dev.S : 1;
    int64_t total_edges = 0;
    for (int r = 0; r < G->dev.R; ++r) total_edges += G->n_edges[r];
    B->cap_dst[1] = max_seeds;
    for (int h = 1; h <= L; ++h) {
        int f = fanouts[L - h];
        int64_t e = (f < 0) ? total_edges : std::min<int64_t>(B->cap_dst[h] * (int64_t)f * S, total_edges);
        B->cap_edges[h] = std::max<int64_t>(e, 1);
        B->cap_dst[h + 1] = std::min<int64_t>(B->cap_dst[h] + B->cap_edges[h], G->total_nodes);
    }
    B->n_words = ceil_div(G->total_nodes, 32);
    // cub temp: max over scans
    size_t cb = 0, t = 0;
    int64_t maxseg = 0;
    for (int h = 1; h <= L; ++h) maxseg = std::max<int64_t>(maxseg, B->cap_dst[h] * S + 1);
    cub::DeviceScan::ExclusiveSum(nullptr, t, (int64_t*)nullptr, (int64_t*)nullptr, (int64_t)maxseg);
    cb = std::max(cb, t);
    if (max_excl > 0) {
        cub::DeviceRadixSort::SortKeys(nullptr, t, (const uint64_t*)nullptr, (uint64_t*)nullptr, (int64_t)(2 * max_excl), 0, 64);
        cb = std::max(cb, t);
        cub::DeviceScan::ExclusiveSum(nullptr, t, (int64_t*)nullptr, (int64_t*)nullptr, (int64_t)(2 * max_excl + 1));
        cb = std::max(cb, t);
    }
    for (int h = 1; h < L; ++h) {
        cub::DeviceRadixSort::SortPairs(nullptr, t, (const int32_t*)nullptr, (int32_t*)nullptr, (const int32_t*)nullptr,
                                        (int32_t*)nullptr, (int64_t)B->cap_edges[h], 0, 31);
        cb = std::max(cb, t);
    }
    B->cub_bytes = cb;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += align_up(bytes > 0 ? bytes : 1);
        return o;
    };
    B->off_err = take(sizeof(int) * 4);
    for (int h = 1; h <= L + 1; ++h) B->off_meta[h <= kMaxL ? h : kMaxL] = 0;
    for (int h = 1; h <= L; ++h) B->off_meta[h] = take(sizeof(HopMeta));
    B->off_seed = take(sizeof(int64_t) * max_seeds);
    for (int h = 1; h <= L; ++h) {
        int64_t nseg = B->cap_dst[h] * S + 1;
        B->off_cnt[h] = take(sizeof(int64_t) * (nseg + kCntMaxBlocks));   // counts, then count_kernel's block totals
        B->off_seg[h] = take(sizeof(int64_t) * nseg);
        B->off_esrcgid[h] = take(sizeof(int64_t) * B->cap_edges[h]);
        B->off_eeid[h] = take(sizeof(int64_t) * B->cap_edges[h]);
        B->off_esrc[h] = take(sizeof(int32_t) * B->cap_edges[h]);
        B->off_segc[h] = take(sizeof(CscSeg) * (nseg - 1 > 0 ? nseg - 1 : 1));
        B->off_tcsr[h] = 0;
        const bool tcsr = getenv("GSB_TCSR") && atoi(getenv("GSB_TCSR")) == 1;   // opt-in (see layer.cu)
        if (tcsr && h < L) {   // layers >= 1 scatter their input gradient through the transposed CSR
            B->off_tcsr[h] = take(sizeof(int32_t) * (5 * B->cap_edges[h] + B->cap_dst[h + 1] + 1));
        }
        B->off_src[h] = take(sizeof(int64_t) * B->cap_dst[h + 1]);
    }
    B->off_map = take(sizeof(int32_t) * G->total_nodes);
    B->off_bitmap = take(sizeof(uint32_t) * B->n_words);
    // word ranks [n_words + 1], then the per-block totals of the rank kernels
    // word ranks, per-block totals, then the fused rank kernel's int64 block flags + epoch + ticket
    B->off_wrank = take(sizeof(int32_t) * (B->n_words + 1 + kRankMaxBlocks) + 8 + sizeof(int64_t) * kRankMaxBlocks + 16);
    B->off_excl = take(sizeof(uint64_t) * (8 * (max_excl > 0 ? max_excl : 1) + 2));
    B->off_cub = take(cb);
    B->total_bytes = off;
    *out = reinterpret_cast<gsb_blocks_t>(B);
    return GSB_OK;
}

gsb_status gsb_blocks_destroy(gsb_blocks_t b) {
    delete reinterpret_cast<Blocks*>(b);
    return GSB_OK;
}

gsb_status gsb_blocks_arena_bytes(gsb_blocks_t b, size_t* bytes) {
    Blocks* B = reinterpret_cast<Blocks*>(b);
    GSB_CHECK_ARG(B && bytes, "null argument");
    *bytes = B->total_bytes;
    return GSB_OK;
}

gsb_status gsb_blocks_init_arena(gsb_blocks_t b, void* arena, size_t arena_bytes, void* stream) {
    Blocks* B = reinterpret_cast<Blocks*>(b);
    GSB_CHECK_ARG(B && arena, "null argument");
    if (arena_bytes < B->total_bytes) {
        set_error("arena %zu < %zu bytes", arena_bytes, B->total_bytes);
        return GSB_EWORKSPACE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    int64_t N = B->g->total_nodes;
    GSB_LAUNCH("init_arena", init_arena_kernel, grid_for(std::max(N, B->n_words), 256, kNumSMs * 8), 256, 0, s,
               at<int32_t>(arena, B->off_map), N, at<uint32_t>(arena, B->off_bitmap), B->n_words,
               at<int>(arena, B->off_err));
    GSB_CUDA(cudaMemsetAsync(rank_flags(B, arena), 0, sizeof(int64_t) * kRankMaxBlocks + 16, s));
    return GSB_OK;
}

gsb_status gsb_sample(gsb_blocks_t b, const gsb_sample_args* a, void* arena, size_t arena_bytes, void* stream) {
    Blocks* B = reinterpret_cast<Blocks*>(b);
    GSB_CHECK_ARG(B && a && arena && a->seeds, "null argument");
    const int64_t* seeds = a->seeds;
    const int64_t n_seeds = a->n_seeds;
    const uint64_t rng_seed = a->rng_seed;
    const int64_t* excl_u = a->excl_u;
    const int64_t* excl_v = a->excl_v;
    const int64_t n_excl = a->n_excl;
    const int32_t excl_etype = a->excl_etype, excl_rev_etype = a->excl_rev_etype;
    GSB_CHECK_ARG(n_seeds >= 1 && n_seeds <= B->max_seeds, "n_seeds %lld out of [1, %lld]", (long long)n_seeds,
                  (long long)B->max_seeds);
    GSB_CHECK_ARG(n_excl >= 0 && n_excl <= B->max_excl, "n_excl %lld exceeds capacity %lld", (long long)n_excl,
                  (long long)B->max_excl);
    GSB_CHECK_ARG(n_excl == 0 || (excl_u && excl_v && excl_etype >= 0 && excl_etype < B->g->dev.R),
                  "bad exclusion arguments");
    GSB_CHECK_ARG(excl_rev_etype < B->g->dev.R, "bad excl_rev_etype");
    if (arena_bytes < B->total_bytes) {
        set_error("arena %zu < %zu bytes", arena_bytes, B->total_bytes);
        return GSB_EWORKSPACE;
    }
    const GraphDev& g = B->g->dev;
    cudaStream_t s = (cudaStream_t)stream;
    const int S = g.S > 0 ? g.S : 1;
    int* err = at<int>(arena, B->off_err);
    int32_t* map = at<int32_t>(arena, B->off_map);
    uint32_t* bitmap = at<uint32_t>(arena, B->off_bitmap);
    int32_t* wrank = at<int32_t>(arena, B->off_wrank);
    void* cub_tmp = at<char>(arena, B->off_cub);

    Excl ex{nullptr, 0, excl_etype, excl_rev_etype >= 0 ? excl_rev_etype : -2, nullptr, nullptr};
    if (n_excl > 0) {
        uint64_t* kin = at<uint64_t>(arena, B->off_excl);
        uint64_t* kout = kin + 2 * B->max_excl;
        int64_t* elo = reinterpret_cast<int64_t*>(kout + 2 * B->max_excl);
        int64_t* ecum = elo + 2 * B->max_excl;
        GSB_LAUNCH("excl_keys", excl_keys_kernel, grid_for(n_excl, 256, 64), 256, 0, s, excl_u, excl_v, n_excl,
                   excl_rev_etype >= 0 ? 1 : 0, kin);
        size_t cb = B->cub_bytes;
        GSB_CUDA(cub::DeviceRadixSort::SortKeys(cub_tmp, cb, kin, kout, (int64_t)(2 * n_excl), 0, 64, s));
        count_launch(16);
        GSB_LAUNCH("excl_ranges", excl_ranges_kernel, grid_for(2 * n_excl + 1, 256, kNumSMs * 4), 256, 0, s, g, kout,
                   2 * n_excl, excl_etype, excl_rev_etype >= 0 ? excl_rev_etype : -2, elo, ecum);
        cb = B->cub_bytes;
        GSB_CUDA(cub::DeviceScan::ExclusiveSum(cub_tmp, cb, ecum, ecum, (int64_t)(2 * n_excl + 1), s));
        count_launch(2);
        ex.keys = kout;
        ex.n = 2 * n_excl;
        ex.lo = elo;
        ex.cum = ecum;
    }

    // err[0] = this sample's latch; err[1] = sticky OR of every earlier sample's latch since the
    // last poll, so an error in any step of a timed loop is still reported afterwards
    if (n_seeds <= 8192) {      // seed_meta_kernel rolls the latch itself
        GSB_LAUNCH("seed_meta", seed_meta_kernel, 1, 1024, 0, s, g, seeds, n_seeds, a->n_seeds_dev,
                   at<int64_t>(arena, B->off_seed), at<HopMeta>(arena, B->off_meta[1]), err);
    } else {
        GSB_LAUNCH("err_roll", err_roll_kernel, 1, 32, 0, s, err);
        HopMeta* m1 = at<HopMeta>(arena, B->off_meta[1]);
        GSB_CUDA(cudaMemsetAsync(m1, 0, sizeof(HopMeta), s));
        GSB_LAUNCH("seed_meta", seed_scan_kernel, grid_for(n_seeds, 256, kNumSMs * 8), 256, 0, s, g, seeds, n_seeds,
                   a->n_seeds_dev, at<int64_t>(arena, B->off_seed), m1, err);
        GSB_LAUNCH("seed_meta_fin", seed_fin_kernel, 1, 32, 0, s, g.T, n_seeds, a->n_seeds_dev, m1, err);
    }
    for (int h = 1; h <= B->L; ++h) {
        HopBufs hb = B->hop(h, arena);
        const int f = B->fanout[B->L - h];
        const int64_t nseg = hb.cap_dst * S;
        if (B->x.first_hop > 0 && h >= B->x.first_hop) {
            gsb_status st = exchange_hop(B, a, hb, h, f, S, rng_seed, map, bitmap, err, cub_tmp, s);
            if (st != GSB_OK) return st;
        } else {
        {
            // count chunks: whole multiples of kCntThreads entries, at most kCntMaxBlocks of them;
            // scan chunks: kScanPerBlock count chunks (whole kCntTile tiles, 16-B aligned)
            const int64_t chunk = ceil_div(ceil_div(nseg + 1, kCntThreads), kCntMaxBlocks) * kCntThreads;
            const int nb = (int)ceil_div(nseg + 1, chunk);
            const int64_t schunk = chunk * kScanPerBlock;
            const int nbs = (int)ceil_div(nseg + 1, schunk);
            int64_t* btot = hb.cnt + nseg + 1;
            GSB_LAUNCH("sample_count", count_kernel, nb, kCntThreads, 0, s, g, hb.meta, hb.dst_gid, hb.cap_dst, f, ex,
                       map, hb.cnt, chunk, btot, err, hb.segc);
            GSB_LAUNCH("sample_scan", count_scan_kernel, nbs, kCntThreads, 0, s, hb.cnt, nseg + 1, schunk, btot, nb,
                       hb.seg_ptr);
        }
        {
            const int G = (f >= 1 && f <= 8) ? 8 : ((f >= 1 && f <= 16) ? 16 : 32);
            const int grid = grid_for(nseg * G, 256, kNumSMs * GSB_FILL_BPS);
            const bool tail = f < 0 || f > kFillCap;
            const int64_t cap = tail ? kFillCap : INT64_MAX;
            if (G == 8)
                GSB_LAUNCH("sample_fill", fill_kernel<8>, grid, 256, 0, s, g, hb.meta, hb.dst_gid, hb.cap_dst,
                           hb.seg_ptr, f, ex, rng_seed, a->step, a->step_dev, h, map, bitmap, hb.e_src_gid, hb.e_eid,
                           err, cap, (const int64_t*)nullptr, 1, 0, (const CscSeg*)hb.segc);
            else if (G == 16)
                GSB_LAUNCH("sample_fill", fill_kernel<16>, grid, 256, 0, s, g, hb.meta, hb.dst_gid, hb.cap_dst,
                           hb.seg_ptr, f, ex, rng_seed, a->step, a->step_dev, h, map, bitmap, hb.e_src_gid, hb.e_eid,
                           err, cap, (const int64_t*)nullptr, 1, 0, (const CscSeg*)hb.segc);
            else
                GSB_LAUNCH("sample_fill", fill_kernel<32>, grid, 256, 0, s, g, hb.meta, hb.dst_gid, hb.cap_dst,
                           hb.seg_ptr, f, ex, rng_seed, a->step, a->step_dev, h, map, bitmap, hb.e_src_gid, hb.e_eid,
                           err, cap, (const int64_t*)nullptr, 1, 0, (const CscSeg*)hb.segc);
            if (tail)
                GSB_LAUNCH("sample_fill_tail", fill_tail_kernel, kNumSMs * 8, 256, 0, s, g, hb.meta, hb.dst_gid,
                           hb.seg_ptr, ex, map, bitmap, hb.e_src_gid, hb.e_eid, err);
        }
        }
        HopMeta* next = (h < B->L) ? at<HopMeta>(arena, B->off_meta[h + 1]) : nullptr;
        {
            const int64_t chunk = ceil_div(ceil_div(B->n_words + 1, kRankTile), kRankMaxBlocks) * kRankTile;
            const int nb = (int)ceil_div(B->n_words + 1, chunk);
            // one launch (rank_fused_kernel) unless GSB_RANK_FUSED=0 (the three-kernel A/B path)
            static const bool fused = !(getenv("GSB_RANK_FUSED") && strcmp(getenv("GSB_RANK_FUSED"), "0") == 0);
            if (fused) {
                GSB_LAUNCH("bitmap_rank", rank_fused_kernel, nb, kRankThreads, 0, s, g, bitmap, B->n_words, chunk, wrank,
                           reinterpret_cast<unsigned long long*>(rank_flags(B, arena)), hb.meta, next, hb.seg_ptr, nseg,
                           hb.cap_src, err);
            } else {
                int32_t* btot = wrank + B->n_words + 1;
                GSB_LAUNCH("bitmap_rank_sum", rank_sum_kernel, nb, kRankThreads, 0, s, bitmap, B->n_words, chunk, btot);
                GSB_LAUNCH("bitmap_rank_scan", rank_scan_kernel, nb, kRankThreads, 0, s, bitmap, B->n_words, chunk,
                           btot, wrank);
                GSB_LAUNCH("hop_meta", hop_meta_kernel, 1, 32, 0, s, g, hb.meta, next, hb.seg_ptr, nseg, bitmap, wrank,
                           hb.cap_src, err);
            }
        }
        GSB_LAUNCH("relabel", relabel_kernel, grid_for(hb.cap_edges, 256, kNumSMs * 8), 256, 0, s, g, hb.meta,
                   hb.e_src_gid, map, bitmap, wrank, hb.e_src);
        if (hb.t_ptr) {
            GSB_LAUNCH("tcsr_prep", tcsr_prep_kernel, grid_for(hb.cap_edges, 256, kNumSMs * 4), 256, 0, s, hb.meta,
                       hb.seg_ptr, S, hb.e_src, hb.cap_edges, hb.e_seg, hb.t_key, hb.t_val);
            size_t cb = B->cub_bytes;
            GSB_CUDA(cub::DeviceRadixSort::SortPairs(cub_tmp, cb, hb.t_key, hb.t_key2, hb.t_val, hb.t_edge,
                                                     (int64_t)hb.cap_edges, 0, 31, s));
            count_launch(8);
            GSB_LAUNCH("tcsr_ptr", tcsr_ptr_kernel, grid_for(hb.cap_src + 1, 256, kNumSMs * 4), 256, 0, s, hb.meta,
                       hb.t_key2, hb.cap_src, hb.t_ptr, hb.t_edge, hb.e_seg, hb.seg_ptr, hb.t_key, hb.t_val);
        }
        GSB_LAUNCH("next_frontier", next_frontier_kernel,
                   grid_for(std::max(hb.cap_dst, B->n_words), 256, kNumSMs * 8), 256, 0, s, g, hb.meta, hb.dst_gid,
                   map, bitmap, wrank, B->n_words, hb.cap_src, hb.src_gid);
    }
    return GSB_OK;
}

gsb_status gsb_block_sizes(gsb_blocks_t b, const void* arena, int32_t layer, int64_t* n_dst, int64_t* n_src,
                                 int64_t* n_edges, int64_t* dst_type_cnt, int64_t* src_type_cnt, void* stream) {
    Blocks* B = reinterpret_cast<Blocks*>(b);
    GSB_CHECK_ARG(B && arena && layer >= 0 && layer < B->L, "bad argument");
    int h = B->hop_of_layer(layer);
    HopMeta m;
    cudaStream_t s = (cudaStream_t)stream;
    GSB_CUDA(cudaMemcpyAsync(&m, at<HopMeta>(const_cast<void*>(arena), B->off_meta[h]), sizeof(HopMeta),
                             cudaMemcpyDeviceToHost, s));
    GSB_CUDA(cudaStreamSynchronize(s));
    if (n_dst) *n_dst = m.n_dst;
    if (n_src) *n_src = m.n_src;
    if (n_edges) *n_edges = m.n_edges;
    for (int t = 0; t < B->g->dev.T; ++t) {
        if (dst_type_cnt) dst_type_cnt[t] = m.dst_off[t + 1] - m.dst_off[t];
        if (src_type_cnt) src_type_cnt[t] = m.src_off[t + 1] - m.src_off[t];
    }
    return GSB_OK;
}

gsb_status gsb_block_view_get(gsb_blocks_t b, const void* arena, int32_t layer, gsb_block_view* out) {
    Blocks* B = reinterpret_cast<Blocks*>(b);
    GSB_CHECK_ARG(B && arena && out && layer >= 0 && layer < B->L, "bad argument");
    HopBufs hb = B->hop(B->hop_of_layer(layer), const_cast<void*>(arena));
    out->dst_gid = hb.dst_gid;
    out->src_gid = hb.src_gid;
    out->seg_ptr = hb.seg_ptr;
    out->e_src_gid = hb.e_src_gid;
    out->e_eid = hb.e_eid;
    out->e_src = hb.e_src;
    out->num_slots = B->g->dev.S > 0 ? B->g->dev.S : 1;
    return GSB_OK;
}

gsb_status gsb_blocks_set_exchange(gsb_blocks_t b, int32_t world, int32_t rank, int32_t first_hop,
                                   const gsb_exchange_bufs* bufs, gsb_exchange_fn fn, void* user) {
    Blocks* B = reinterpret_cast<Blocks*>(b);
    GSB_CHECK_ARG(B && (first_hop == 0 || (bufs && fn)), "null argument");
    GSB_CHECK_ARG(world >= 1 && world <= kMaxPeers && rank >= 0 && rank < world, "bad world / rank");
    GSB_CHECK_ARG(first_hop >= 0 && first_hop <= B->L, "first_hop %d out of [0, %d]", first_hop, B->L);
    memset(&B->x, 0, sizeof(Xchg));
    if (first_hop == 0) return GSB_OK;
    B->x.world = world;
    B->x.rank = rank;
    B->x.first_hop = first_hop;
    B->x.req_send = bufs->req_send;
    B->x.req_perm = bufs->req_perm;
    B->x.send_cnt = bufs->send_cnt;
    B->x.cursor = bufs->cursor;
    B->x.req_recv = bufs->req_recv;
    B->x.cap_recv = bufs->cap_recv;
    B->x.xoff = bufs->xoff;
    B->x.srv_meta = reinterpret_cast<HopMeta*>(bufs->srv_meta);
    B->x.srv_cnt = bufs->srv_cnt;
    B->x.srv_seg = bufs->srv_seg;
    B->x.srv_gid = bufs->srv_gid;
    B->x.srv_eid = bufs->srv_eid;
    B->x.cap_srv_e = bufs->cap_srv_e;
    B->x.srv_wcnt = bufs->srv_wcnt;
    B->x.resp_cnt = bufs->resp_cnt;
    B->x.resp_seg = bufs->resp_seg;
    B->x.resp_gid = bufs->resp_gid;
    B->x.resp_eid = bufs->resp_eid;
    B->x.cap_resp_e = bufs->cap_resp_e;
    B->x.fn = fn;
    B->x.user = user;
    return GSB_OK;
}

gsb_status gsb_exchange_sizes(gsb_blocks_t b, int32_t world, int64_t* cap_dst, int64_t* cap_recv,
                              int64_t* cap_srv_e, int64_t* cap_resp_e, int64_t* srv_cnt_len, int64_t* meta_bytes) {
    Blocks* B = reinterpret_cast<Blocks*>(b);
    GSB_CHECK_ARG(B && cap_dst && cap_recv && cap_srv_e && cap_resp_e && srv_cnt_len && meta_bytes, "null argument");
    GSB_CHECK_ARG(world >= 1 && world <= kMaxPeers, "bad world");
    const int S = B->g->dev.S > 0 ? B->g->dev.S : 1;
    int64_t cd = 0, ce = 0, fmax = 1;
    for (int h = 1; h <= B->L; ++h) {
        cd = std::max(cd, B->cap_dst[h]);
        ce = std::max(ce, B->cap_edges[h]);
        fmax = std::max<int64_t>(fmax, B->fanout[B->L - h]);
    }
    *cap_dst = cd;
    *cap_recv = cd * world;                 // every rank may ask this one for its whole frontier
    *cap_srv_e = cd * world * S * fmax;
    *cap_resp_e = ce;
    *srv_cnt_len = cd * world * S + 1 + kCntMaxBlocks;
    *meta_bytes = sizeof(HopMeta);
    return GSB_OK;
}

gsb_status gsb_blocks_poll_error(gsb_blocks_t b, void* arena, int32_t* code, void* stream) {
    Blocks* B = reinterpret_cast<Blocks*>(b);
    GSB_CHECK_ARG(B && arena && code, "null argument");
    cudaStream_t s = (cudaStream_t)stream;
    int hw[2] = {0, 0};
    int* err = at<int>(arena, B->off_err);
    GSB_CUDA(cudaMemcpyAsync(hw, err, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
    GSB_CUDA(cudaMemsetAsync(err + 1, 0, sizeof(int), s));      // the sticky word restarts
    GSB_CUDA(cudaStreamSynchronize(s));
    const int h = hw[0] ? hw[0] : hw[1];
    *code = h;
    if (h != 0) {
        set_error("device-side error %d latched during sampling", h);
        return GSB_EDEVICE;
    }
    return GSB_OK;
}

gsb_status gsb_blocks_input_rows(gsb_blocks_t b, int64_t* max_rows) {
    Blocks* B = reinterpret_cast<Blocks*>(b);
    GSB_CHECK_ARG(B && max_rows, "null argument");
    *max_rows = B->cap_dst[B->L + 1];
    return GSB_OK;
}

gsb_status gsb_blocks_dst_rows(gsb_blocks_t b, int32_t layer, int64_t* max_rows) {
    Blocks* B = reinterpret_cast<Blocks*>(b);
    GSB_CHECK_ARG(B && max_rows && layer >= 0 && layer < B->L, "bad argument");
    *max_rows = B->cap_dst[B->hop_of_layer(layer)];
    return GSB_OK;
}

gsb_status gsb_gather_block_inputs(gsb_blocks_t b, const void* arena, void* out, void* stream) {
    Blocks* B = reinterpret_cast<Blocks*>(b);
    GSB_CHECK_ARG(B && arena && out, "null argument");
    const Graph* G = B->g;
    GSB_CHECK_ARG(G->dev.feat_dim > 0, "features not registered (or not one width for all ntypes)");
    HopBufs hb = B->hop(B->L, const_cast<void*>(arena));
    return launch_gather(G, hb.src_gid, &hb.meta->n_src, 0, hb.cap_src, out, (cudaStream_t)stream);
}

}  // extern "C"
