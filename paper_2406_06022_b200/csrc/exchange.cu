// exchange.cu -- node-ID partitioning of the feature store across GPUs (SURVEY §8(e), §2.4
// C4/C5): owner bucketing of requested gids (K11), gather from the local shard on the owner,
// and unpacking of the returned rows.  The collectives themselves (NCCL all-to-all) are issued
// by the caller between these calls.  Contract: include/gsb.h "Partitioned feature store".
#include <cub/device/device_scan.cuh>

#include "gsb_internal.cuh"

namespace gsb {

struct PartDev {
    int32_t world, rank, T;
    int64_t lo[kMaxT][9];   // local-id boundaries of each rank per ntype (world <= 8)
    int64_t node_off[kMaxT + 1];
    const char* shard[kMaxT];    // local shard rows [lo[t][rank], lo[t][rank+1])
    int32_t dim, row_bytes;      // elements / bytes per row (fp32 or bf16)
};

__device__ __forceinline__ int part_type(const PartDev& p, int64_t gid) {
    int t = 0;
    for (int k = 1; k < p.T; ++k) t += (gid >= p.node_off[k]) ? 1 : 0;
    return t;
}
__device__ __forceinline__ int part_owner(const PartDev& p, int t, int64_t local) {
    int r = 0;
    for (int k = 1; k < p.world; ++k) r += (local >= p.lo[t][k]) ? 1 : 0;
    return r;
}

// Warp-aggregated: one shared-memory atomic per (warp, owner) instead of one per id.
__global__ void owner_count_kernel(PartDev p, const int64_t* __restrict__ gid, const int64_t* __restrict__ n_dev,
                                   int64_t n_cap, unsigned long long* __restrict__ cnt) {
    GSB_PDL_ENTRY();
    __shared__ unsigned long long sc[8];
    if (threadIdx.x < 8) sc[threadIdx.x] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t n = n_dev ? min(*n_dev, n_cap) : n_cap;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x; b < n; b += stride) {
        const int64_t i = b + threadIdx.x;
        int w = -1;
        if (i < n) {
            const int64_t x = gid[i];
            const int t = part_type(p, x);
            w = part_owner(p, t, x - p.node_off[t]);
        }
        for (int o = 0; o < p.world; ++o) {
            const unsigned bal = __ballot_sync(0xffffffffu, w == o);
            if (lane == 0 && bal) atomicAdd(&sc[o], (unsigned long long)__popc(bal));
        }
    }
    __syncthreads();
    if (threadIdx.x < p.world && sc[threadIdx.x]) atomicAdd(&cnt[threadIdx.x], sc[threadIdx.x]);
}

// cursor[w] counts positions handed out inside owner w's bucket; one global atomic per
// (warp, owner), lanes take consecutive slots by their rank inside the ballot.  The order
// inside a bucket does not affect the result: perm maps every row back.
__global__ void owner_scatter_kernel(PartDev p, const int64_t* __restrict__ gid, const int64_t* __restrict__ n_dev,
                                     int64_t n_cap, const unsigned long long* __restrict__ cnt,
                                     unsigned long long* __restrict__ cursor, int64_t* __restrict__ send_gid,
                                     int32_t* __restrict__ perm) {
    GSB_PDL_ENTRY();
    __shared__ unsigned long long base[8];
    if (threadIdx.x == 0) {
        unsigned long long a = 0;
        for (int w = 0; w < p.world; ++w) {
            base[w] = a;
            a += cnt[w];
        }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    const int64_t n = n_dev ? min(*n_dev, n_cap) : n_cap;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x; b < n; b += stride) {
        const int64_t i = b + threadIdx.x;
        int w = -1;
        int64_t x = 0;
        if (i < n) {
            x = gid[i];
            const int t = part_type(p, x);
            w = part_owner(p, t, x - p.node_off[t]);
        }
        for (int o = 0; o < p.world; ++o) {
            const unsigned bal = __ballot_sync(0xffffffffu, w == o);
            if (!bal) continue;
            const int leader = __ffs(bal) - 1;
            unsigned long long start = 0;
            if (lane == leader) start = atomicAdd(&cursor[o], (unsigned long long)__popc(bal));
            start = __shfl_sync(0xffffffffu, start, leader);
            if (w == o) {
                const int64_t pos = (int64_t)(base[o] + start + __popc(bal & lt));
                send_gid[pos] = x;
                perm[i] = (int32_t)pos;
            }
        }
    }
}

// row copies in 16-byte chunks (dtype-agnostic)
__global__ void shard_gather_kernel(PartDev p, const int64_t* __restrict__ gid, int64_t n, uint4* __restrict__ out) {
    GSB_PDL_ENTRY();
    const int d16 = p.row_bytes >> 4;
    const int64_t total = n * d16;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i / d16;
        const int c = (int)(i - row * d16);
        const int64_t x = gid[row];
        const int t = part_type(p, x);
        const int64_t local = x - p.node_off[t] - p.lo[t][p.rank];
        out[i] = __ldg(reinterpret_cast<const uint4*>(p.shard[t] + local * p.row_bytes) + c);
    }
}

__global__ void rows_permute_kernel(const char* __restrict__ rows, int row_bytes, const int32_t* __restrict__ perm,
                                    const int64_t* __restrict__ n_dev, int64_t n_cap, uint4* __restrict__ out) {
    GSB_PDL_ENTRY();
    const int64_t n = n_dev ? min(*n_dev, n_cap) : n_cap;
    const int d16 = row_bytes >> 4;
    const int64_t total = n * d16;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = i / d16;
        const int c = (int)(i - row * d16);
        out[i] = __ldg(reinterpret_cast<const uint4*>(rows + (int64_t)perm[row] * row_bytes) + c);
    }
}

struct Part {
    PartDev dev;
};

}  // namespace gsb

using namespace gsb;

extern "C" {

gsb_status gsb_partition_create(int32_t num_ntypes, const int64_t* ntype_count, int32_t world, int32_t rank,
                                const int64_t* bounds, gsb_partition_t* out) {
    GSB_CHECK_ARG(out && ntype_count && bounds, "null argument");
    GSB_CHECK_ARG(num_ntypes >= 1 && num_ntypes <= kMaxT, "bad num_ntypes");
    GSB_CHECK_ARG(world >= 1 && world <= 8 && rank >= 0 && rank < world, "world %d / rank %d unsupported", world, rank);
    Part* P = new Part();
    memset(&P->dev, 0, sizeof(PartDev));
    P->dev.world = world;
    P->dev.rank = rank;
    P->dev.T = num_ntypes;
    P->dev.node_off[0] = 0;
    for (int t = 0; t < num_ntypes; ++t) {
        P->dev.node_off[t + 1] = P->dev.node_off[t] + ntype_count[t];
        for (int w = 0; w <= world; ++w) P->dev.lo[t][w] = bounds[t * (world + 1) + w];
        if (P->dev.lo[t][0] != 0 || P->dev.lo[t][world] != ntype_count[t]) {
            delete P;
            set_error("bounds of ntype %d must span [0, %lld]", t, (long long)ntype_count[t]);
            return GSB_EINVAL;
        }
    }
    for (int t = num_ntypes + 1; t <= kMaxT; ++t) P->dev.node_off[t] = P->dev.node_off[num_ntypes];
    *out = reinterpret_cast<gsb_partition_t>(P);
    return GSB_OK;
}

gsb_status gsb_partition_destroy(gsb_partition_t p) {
    delete reinterpret_cast<Part*>(p);
    return GSB_OK;
}

gsb_status gsb_partition_set_shard(gsb_partition_t p, int32_t ntype, const void* rows, int32_t dim, int32_t dtype) {
    Part* P = reinterpret_cast<Part*>(p);
    const int es = dtype_size(dtype);
    GSB_CHECK_ARG(P && ntype >= 0 && ntype < P->dev.T && es > 0 && dim > 0 && (dim * es) % 16 == 0,
                  "bad argument (rows must be a positive multiple of 16 bytes)");
    GSB_CHECK_ARG(P->dev.dim == 0 || P->dev.row_bytes == dim * es, "all shards must share one row format");
    GSB_CHECK_ARG(((uintptr_t)rows & 15) == 0, "shard must be 16-byte aligned");
    P->dev.dim = dim;
    P->dev.row_bytes = dim * es;
    P->dev.shard[ntype] = static_cast<const char*>(rows);
    return GSB_OK;
}

gsb_status gsb_bucket_by_owner(gsb_partition_t p, const int64_t* gid, const int64_t* n_dev, int64_t n_cap,
                               int64_t* send_gid, int32_t* perm, int64_t* send_counts, void* ws, void* stream) {
    Part* P = reinterpret_cast<Part*>(p);
    GSB_CHECK_ARG(P && gid && send_gid && perm && send_counts && ws && n_cap >= 0, "null argument");
    cudaStream_t s = (cudaStream_t)stream;
    unsigned long long* cnt = reinterpret_cast<unsigned long long*>(send_counts);
    unsigned long long* cursor = reinterpret_cast<unsigned long long*>(ws);
    GSB_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * P->dev.world, s));
    GSB_CUDA(cudaMemsetAsync(cursor, 0, sizeof(int64_t) * P->dev.world, s));
    if (n_cap == 0) return GSB_OK;
    const int grid = grid_for(n_cap, 256, kNumSMs * 4);
    GSB_LAUNCH("owner_count", owner_count_kernel, grid, 256, 0, s, P->dev, gid, n_dev, n_cap, cnt);
    GSB_LAUNCH("owner_scatter", owner_scatter_kernel, grid, 256, 0, s, P->dev, gid, n_dev, n_cap, cnt, cursor,
               send_gid, perm);
    return GSB_OK;
}

gsb_status gsb_shard_gather(gsb_partition_t p, const int64_t* gid, int64_t n, void* out, void* stream) {
    Part* P = reinterpret_cast<Part*>(p);
    GSB_CHECK_ARG(P && (n == 0 || (gid && out)), "null argument");
    GSB_CHECK_ARG(P->dev.dim > 0, "no shard registered");
    for (int t = 0; t < P->dev.T; ++t)
        GSB_CHECK_ARG(P->dev.shard[t] || P->dev.lo[t][P->dev.rank + 1] == P->dev.lo[t][P->dev.rank],
                      "shard of ntype %d not registered", t);
    if (n == 0) return GSB_OK;
    GSB_LAUNCH("shard_gather", shard_gather_kernel, grid_for(n * (P->dev.row_bytes / 16), 256, kNumSMs * 8), 256, 0,
               (cudaStream_t)stream, P->dev, gid, n, static_cast<uint4*>(out));
    return GSB_OK;
}

gsb_status gsb_rows_permute(const void* rows, int32_t row_bytes, const int32_t* perm, const int64_t* n_dev,
                            int64_t n_cap, void* out, void* stream) {
    GSB_CHECK_ARG(rows && perm && out && row_bytes > 0 && row_bytes % 16 == 0 && n_cap >= 0, "bad argument");
    if (n_cap == 0) return GSB_OK;
    GSB_LAUNCH("rows_permute", rows_permute_kernel, grid_for(n_cap * (row_bytes / 16), 256, kNumSMs * 8), 256, 0,
               (cudaStream_t)stream, static_cast<const char*>(rows), row_bytes, perm, n_dev, n_cap,
               static_cast<uint4*>(out));
    return GSB_OK;
}

}  // extern "C"
