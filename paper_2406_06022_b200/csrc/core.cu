// core.cu -- errors, instrumentation, graph store (CSC build on the device), feature
// gather, Adam.  See include/gsb.h for the contract of every extern "C" entry point.
#include <stdarg.h>

#include <cub/device/device_radix_sort.cuh>
#include <atomic>
#include <cstring>
#include <mutex>

#include <nvtx3/nvToolsExt.h>

#include "gemm_tma3.cuh"
#include "umma.cuh"
#include "gsb_internal.cuh"

namespace gsb {

static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};
static bool g_prof_on = false;
struct ProfRec {
    const char* name;
    cudaEvent_t a, b;
    cudaStream_t s;
};
static std::vector<ProfRec> g_prof;
static std::vector<cudaEvent_t> g_event_pool;
static std::mutex g_prof_mu;
static thread_local const char* g_pending_name = nullptr;
static thread_local cudaEvent_t g_pending_ev = nullptr;

void set_error(const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
}

gsb_status cuda_status(cudaError_t e, const char* what) {
    set_error("CUDA error in %s: %s", what, cudaGetErrorString(e));
    return GSB_ECUDA;
}

void count_launch(int n) { g_launches += n; }

static cudaEvent_t get_event() {
    if (!g_event_pool.empty()) {
        cudaEvent_t e = g_event_pool.back();
        g_event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

// Every launch sits in an NVTX range named after the kernel's role (rgcn_agg_l0,
// sample_fill, ...): ncu --nvtx --print-nvtx-rename kernel reports launches by these names.
// Without an attached tool the NVTX calls are no-ops.
// GSB_DEBUG_SYNC=1 (tools): synchronize after every eager launch and report the failing
// kernel by name (device faults otherwise surface at a later, unrelated call)
static thread_local const char* t_last_launch = nullptr;
static bool debug_sync() {
    static int on = -1;
    if (on < 0) on = getenv("GSB_DEBUG_SYNC") ? 1 : 0;
    return on == 1;
}

void prof_begin(const char* name, cudaStream_t s) {
    nvtxRangePushA(name);
    t_last_launch = name;
    if (!g_prof_on) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_pending_name = name;
    g_pending_ev = get_event();
    cudaEventRecord(g_pending_ev, s);
}

void prof_end(cudaStream_t s) {
    nvtxRangePop();
    if (debug_sync()) {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(s, &cs);
        if (cs == cudaStreamCaptureStatusNone) {
            const cudaError_t e = cudaStreamSynchronize(s);
            if (e != cudaSuccess)
                fprintf(stderr, "[gsb] kernel %s failed: %s\n", t_last_launch ? t_last_launch : "?", cudaGetErrorString(e));
        }
    }
    if (!g_prof_on || !g_pending_name) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    cudaEvent_t b = get_event();
    cudaEventRecord(b, s);
    g_prof.push_back({g_pending_name, g_pending_ev, b, s});
    g_pending_name = nullptr;
}

// ------------------------------------------------------------------------------------
// CSC build kernels
// ------------------------------------------------------------------------------------
// keys (dst - dst_lo, src) of the kept edges whose dst lies in [dst_lo, dst_hi) (the whole
// range for a plain build); n_kept[1] counts the kept edges with dst < dst_lo (the global CSC
// position of a partition's first edge)
__global__ void csc_keys_kernel(const int32_t* __restrict__ src, const int32_t* __restrict__ dst,
                                const uint8_t* __restrict__ keep, int64_t n, int64_t dst_lo, int64_t dst_hi,
                                uint64_t* __restrict__ keys, unsigned long long* __restrict__ n_kept) {
    GSB_PDL_ENTRY();
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    unsigned long long local = 0, before = 0;
    for (; i < n; i += stride) {
        const bool k = keep ? (keep[i] != 0) : true;
        const int64_t d = dst[i];
        const bool in = k && d >= dst_lo && d < dst_hi;
        keys[i] = in ? (((uint64_t)(d - dst_lo) << 32) | (uint32_t)src[i]) : ~0ull;
        local += in ? 1 : 0;
        before += (k && d < dst_lo) ? 1 : 0;
    }
    for (int o = 16; o > 0; o >>= 1) {
        local += __shfl_xor_sync(0xffffffffu, local, o);
        before += __shfl_xor_sync(0xffffffffu, before, o);
    }
    if ((threadIdx.x & 31) == 0 && local) atomicAdd(n_kept, local);
    if ((threadIdx.x & 31) == 0 && before) atomicAdd(n_kept + 1, before);
}

__global__ void csc_finish_kernel(const uint64_t* __restrict__ keys, const unsigned long long* __restrict__ n_kept_p,
                                  int64_t n_dst, int64_t* __restrict__ indptr, int32_t* __restrict__ indices) {
    GSB_PDL_ENTRY();
    const int64_t n_kept = (int64_t)*n_kept_p;
    int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_kept; i += stride)
        indices[i] = (int32_t)(uint32_t)(keys[i] & 0xffffffffull);
    for (int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; v <= n_dst; v += stride) {
        uint64_t key = (uint64_t)v << 32;
        int64_t lo = 0, hi = n_kept;
        while (lo < hi) {
            int64_t m = (lo + hi) >> 1;
            if (keys[m] < key) lo = m + 1; else hi = m;
        }
        indptr[v] = lo;
    }
}

// ------------------------------------------------------------------------------------
// gather: out[i, :] = F_t[gid_i - off_t, :]; one 16-byte chunk per thread-iteration
// (dtype-agnostic exact copy: fp32 or bf16 rows)
// ------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) gather_kernel(GraphDev g, const int64_t* __restrict__ gid,
                                                     const int64_t* __restrict__ n_dev, int64_t n_host,
                                                     uint4* __restrict__ out) {
    GSB_PDL_ENTRY();
    const int64_t n = n_dev ? *n_dev : n_host;
    const int d16 = g.feat_row_bytes >> 4;
    const int64_t total = n * d16;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t N = g.node_off[g.T];
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    // 4 independent rows in flight per thread
    for (; i < total; i += 4 * stride) {
        uint4 v[4];
        int64_t idx[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            idx[u] = i + u * stride;
            v[u] = make_uint4(0u, 0u, 0u, 0u);
            if (idx[u] < total) {
                int64_t row = idx[u] / d16;
                int c = (int)(idx[u] - row * d16);
                int64_t x = __ldg(gid + row);
                if (x >= 0 && x < N) v[u] = ldg_nc_u4(feat_row(g, x) + c);
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (idx[u] < total) out[idx[u]] = v[u];
    }
}

// 32-byte chunks (256-bit loads, LDG.E.ENL2.256): half the address work and load instructions
// per byte of the 16-byte kernel; 8 chunks of different rows in flight per thread.  Used for
// rows that are a multiple of 32 bytes (every config's 64-d fp32 / 128-d bf16 rows).
__global__ void __launch_bounds__(256) gather32_kernel(GraphDev g, const int64_t* __restrict__ gid,
                                                       const int64_t* __restrict__ n_dev, int64_t n_host,
                                                       uint4* __restrict__ out) {
    GSB_PDL_ENTRY();
    constexpr int U = 8;
    const int64_t n = n_dev ? *n_dev : n_host;
    const int d32 = g.feat_row_bytes >> 5;
    const int64_t total = n * d32;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t N = g.node_off[g.T];
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += U * stride) {
        uint32_t v[U][8];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t idx = i + u * stride;
#pragma unroll
            for (int k = 0; k < 8; ++k) v[u][k] = 0u;
            if (idx < total) {
                const int64_t row = idx / d32;
                const int c = (int)(idx - row * d32);
                const int64_t x = __ldg(gid + row);
                if (x >= 0 && x < N) {
                    const char* p = reinterpret_cast<const char*>(feat_row(g, x)) + 32 * c;
                    asm volatile("ld.global.nc.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                                 : "=r"(v[u][0]), "=r"(v[u][1]), "=r"(v[u][2]), "=r"(v[u][3]), "=r"(v[u][4]),
                                   "=r"(v[u][5]), "=r"(v[u][6]), "=r"(v[u][7])
                                 : "l"(p));
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t idx = i + u * stride;
            if (idx < total) {
                out[2 * idx] = make_uint4(v[u][0], v[u][1], v[u][2], v[u][3]);
                out[2 * idx + 1] = make_uint4(v[u][4], v[u][5], v[u][6], v[u][7]);
            }
        }
    }
}

gsb_status launch_gather(const Graph* G, const int64_t* gid, const int64_t* n_dev, int64_t n_host, int64_t n_max,
                         void* out, cudaStream_t s) {
    static const bool g16 = getenv("GSB_GATHER16") != nullptr;     // A/B knob
    if (!g16 && G->dev.feat_row_bytes % 32 == 0) {
        // bounded grid: the unique-row fetch is latency / NVLink bound and runs beside the compute
        // phase's GEMMs (one CTA per SM); 2 blocks per SM keep ~4 MB in flight
        const int64_t work = n_max * (G->dev.feat_row_bytes / 32);
        static const int bps = getenv("GSB_GATHER_BPS") ? atoi(getenv("GSB_GATHER_BPS")) : 2;   // A/B knob
        const int grid = grid_for(ceil_div(work, 8), 256, kNumSMs * bps);
        GSB_LAUNCH("gather", gather32_kernel, grid, 256, 0, s, G->dev, gid, n_dev, n_host, static_cast<uint4*>(out));
        return GSB_OK;
    }
    int64_t work = n_max * (G->dev.feat_row_bytes / 16);
    int grid = grid_for(ceil_div(work, 4), 256, kNumSMs * 8);
    GSB_LAUNCH("gather", gather_kernel, grid, 256, 0, s, G->dev, gid, n_dev, n_host, static_cast<uint4*>(out));
    return GSB_OK;
}

// ------------------------------------------------------------------------------------
// Adam (bias-corrected), float4 vectorised
// ------------------------------------------------------------------------------------
// hi / lo (optional): the 3xTF32 split of the updated parameters (hi = rna_tf32(p), lo =
// rna_tf32(p - hi)) for the GEMMs' weight images, written in the same pass
__device__ __forceinline__ void adam_split(float x, float* hi, float* lo, int64_t i) {
    uint32_t h, l;
    umma::split_tf32(x, h, l);
    hi[i] = __uint_as_float(h);
    lo[i] = __uint_as_float(l);
}
// pad: one parameter segment [off, off + rows*cols) whose split is also written with a padded
// row stride (ld) into pad_hi / pad_lo (a weight whose own row stride is not 16-B aligned)
struct AdamPad {
    int64_t off;
    int32_t rows, cols, ld;
    float *hi, *lo;
};
__device__ __forceinline__ void adam_pad(const AdamPad& pd, int64_t i, uint32_t h, uint32_t l) {
    const int64_t q = i - pd.off;
    if (q < 0 || q >= (int64_t)pd.rows * pd.cols) return;
    const uint32_t r = (uint32_t)q / (uint32_t)pd.cols;
    const int64_t o = (int64_t)r * pd.ld + ((uint32_t)q - r * (uint32_t)pd.cols);
    pd.hi[o] = __uint_as_float(h);
    pd.lo[o] = __uint_as_float(l);
}
__global__ void __launch_bounds__(256) adam_kernel(float* __restrict__ p, const float* __restrict__ gr,
                                                   float* __restrict__ m, float* __restrict__ v, int64_t n, float lr,
                                                   float b1, float b2, float eps, float c1, float c2,
                                                   const int32_t* __restrict__ t_dev, float* __restrict__ hi,
                                                   float* __restrict__ lo, AdamPad pd) {
    GSB_PDL_ENTRY();
    __shared__ float sc[2];
    if (t_dev) {   // bias corrections from the device step counter (graph replay), once per block
        if (threadIdx.x == 0) {
            const float t = (float)*t_dev;
            sc[0] = 1.f - powf(b1, t);
            sc[1] = 1.f - powf(b2, t);
        }
        __syncthreads();
        c1 = sc[0];
        c2 = sc[1];
    }
    const float a1 = lr / c1, r2 = 1.f / c2;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t n4 = n >> 2;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
        float4 g = reinterpret_cast<const float4*>(gr)[i];
        float4 mi = reinterpret_cast<float4*>(m)[i];
        float4 vi = reinterpret_cast<float4*>(v)[i];
        float4 pi = reinterpret_cast<float4*>(p)[i];
#define ADAM1(c)                                         \
        mi.c = b1 * mi.c + (1.f - b1) * g.c;             \
        vi.c = b2 * vi.c + (1.f - b2) * g.c * g.c;       \
        pi.c -= a1 * mi.c / (sqrtf(vi.c * r2) + eps);
        ADAM1(x) ADAM1(y) ADAM1(z) ADAM1(w)
#undef ADAM1
        reinterpret_cast<float4*>(m)[i] = mi;
        reinterpret_cast<float4*>(v)[i] = vi;
        reinterpret_cast<float4*>(p)[i] = pi;
        if (hi) {
            uint32_t h0, h1, h2, h3, l0, l1, l2, l3;
            umma::split_tf32(pi.x, h0, l0);
            umma::split_tf32(pi.y, h1, l1);
            umma::split_tf32(pi.z, h2, l2);
            umma::split_tf32(pi.w, h3, l3);
            reinterpret_cast<uint4*>(hi)[i] = make_uint4(h0, h1, h2, h3);
            reinterpret_cast<uint4*>(lo)[i] = make_uint4(l0, l1, l2, l3);
            if (pd.hi && 4 * i + 3 >= pd.off && 4 * i < pd.off + (int64_t)pd.rows * pd.cols) {
                adam_pad(pd, 4 * i, h0, l0);
                adam_pad(pd, 4 * i + 1, h1, l1);
                adam_pad(pd, 4 * i + 2, h2, l2);
                adam_pad(pd, 4 * i + 3, h3, l3);
            }
        }
    }
    for (int64_t i = 4 * n4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride) {
        const float g = gr[i];
        const float mi = b1 * m[i] + (1.f - b1) * g;
        const float vi = b2 * v[i] + (1.f - b2) * g * g;
        m[i] = mi;
        v[i] = vi;
        p[i] -= a1 * mi / (sqrtf(vi * r2) + eps);
        if (hi) {
            adam_split(p[i], hi, lo, i);
            if (pd.hi) adam_pad(pd, i, __float_as_uint(hi[i]), __float_as_uint(lo[i]));
        }
    }
}

__global__ void counter_add_kernel(int32_t* c, int32_t d) {
    GSB_PDL_ENTRY(); *c += d; }

__global__ void spin_kernel(int64_t ns) {
    GSB_PDL_ENTRY();
    uint64_t t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    } while ((int64_t)(t1 - t0) < ns);
}

gsb_status set_feature_format(Graph* G, int32_t ntype, int32_t dim, int32_t dtype) {
    const int es = dtype_size(dtype);
    GSB_CHECK_ARG(es > 0, "dtype %d not GSB_F32 / GSB_BF16", dtype);
    GSB_CHECK_ARG(dim > 0 && (dim * es) % 16 == 0, "feature rows must be a positive multiple of 16 bytes "
                  "(dim %d x %d B)", dim, es);
    GSB_CHECK_ARG(!G->dtype_set || G->dev.feat_dtype == dtype, "all ntypes must share one feature dtype");
    G->dtype_set = true;
    G->dev.feat_dtype = dtype;
    G->dev.dim_t[ntype] = dim;
    G->dev.row_bytes_t[ntype] = dim * es;
    // uniform width over the registered ntypes (required by the fused layer-0 path and gathers)
    int u = 0;
    for (int t = 0; t < G->dev.T; ++t) {
        if (!G->dev.dim_t[t]) continue;
        u = (u == 0 || u == G->dev.dim_t[t]) ? G->dev.dim_t[t] : -1;
    }
    G->dev.feat_dim = u > 0 ? u : 0;
    G->dev.feat_row_bytes = u > 0 ? u * es : 0;
    return GSB_OK;
}

}  // namespace gsb

using namespace gsb;

// ====================================================================================
// extern "C" entry points
// ====================================================================================
namespace gsb {
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = getenv("GSB_PDL");   // opt-in: measured neutral to -4 % under CUDA graphs
        return e && atoi(e) != 0;
    }();
    return on;
}

namespace {
struct ForkState {
    bool init = false, enabled = true;
    cudaStream_t side = nullptr;
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
};
ForkState g_fork[16];
}  // namespace

cudaStream_t fork_begin(cudaStream_t s) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 16) return s;
    ForkState& f = g_fork[dev];
    if (!f.init) {
        f.init = true;
        const char* e = getenv("GSB_NO_FORK");
        f.enabled = !(e && atoi(e) != 0) &&
                    cudaStreamCreateWithFlags(&f.side, cudaStreamNonBlocking) == cudaSuccess &&
                    cudaEventCreateWithFlags(&f.ev_fork, cudaEventDisableTiming) == cudaSuccess &&
                    cudaEventCreateWithFlags(&f.ev_join, cudaEventDisableTiming) == cudaSuccess;
    }
    if (!f.enabled) return s;
    if (cudaEventRecord(f.ev_fork, s) != cudaSuccess || cudaStreamWaitEvent(f.side, f.ev_fork, 0) != cudaSuccess)
        return s;
    return f.side;
}

gsb_status fork_end(cudaStream_t s, cudaStream_t side) {
    if (side == s) return GSB_OK;
    int dev = 0;
    GSB_CUDA(cudaGetDevice(&dev));
    ForkState& f = g_fork[dev];
    GSB_CUDA(cudaEventRecord(f.ev_join, side));
    GSB_CUDA(cudaStreamWaitEvent(s, f.ev_join, 0));
    return GSB_OK;
}

// ------------------------------------------------------------------------------------
// TMA tensor maps (gemm_tma.cuh): cuTensorMapEncodeTiled through the runtime's driver entry
// point (no libcuda link dependency)
// ------------------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

bool encode_tmap_f32(CUtensorMap* m, const float* base, int64_t width, int64_t rows, int64_t ld, int box_w,
                     int box_h, bool swz128) {
    EncodeTiledFn fn = encode_fn();
    if (!fn || width < 1 || rows < 1) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)width, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(float)};
    const cuuint32_t box[2] = {(cuuint32_t)box_w, (cuuint32_t)box_h};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE,
                          swz128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool encode_tmap_bf16_2d(CUtensorMap* m, const void* base, int64_t width, int64_t rows, int64_t ld, int box_w,
                         int box_h) {
    EncodeTiledFn fn = encode_fn();
    if (!fn || width < 1 || rows < 1) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)width, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
    const cuuint32_t box[2] = {(cuuint32_t)box_w, (cuuint32_t)box_h};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool encode_tmap_nd(CUtensorMap* m, const float* base, int rank, const int64_t* dims, const int64_t* strides,
                    const int* box, int swizzle) {
    EncodeTiledFn fn = encode_fn();
    if (!fn || rank < 2 || rank > 3) return false;
    cuuint64_t d[3], st[2];
    cuuint32_t b[3], es[3] = {1, 1, 1};
    for (int i = 0; i < rank; ++i) {
        if (dims[i] < 1) return false;
        d[i] = (cuuint64_t)dims[i];
        b[i] = (cuuint32_t)box[i];
    }
    for (int i = 0; i < rank - 1; ++i) st[i] = (cuuint64_t)strides[i] * sizeof(float);
    const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, (cuuint32_t)rank, const_cast<float*>(base), d, st, b, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, (CUtensorMapSwizzle)swizzle,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

}  // namespace gsb

extern "C" {

const char* gsb_last_error(void) { return g_err.c_str(); }
int32_t gsb_version(void) { return 100; }
int64_t gsb_launch_count(void) { return g_launches.load(); }

gsb_status gsb_profile_enable(int32_t on) {
    g_prof_on = on != 0;
    return GSB_OK;
}

// one line per profiled launch, in enqueue order: name, stream index (order of first use),
// start and duration in us relative to the earliest launch start (tools: step timelines)
gsb_status gsb_profile_timeline(char* buf, size_t buflen) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    GSB_CUDA(cudaDeviceSynchronize());
    std::string out;
    if (!g_prof.empty()) {
        std::vector<cudaStream_t> streams;
        float t0 = 0.f;
        for (auto& r : g_prof) {
            float t = 0.f;
            cudaEventElapsedTime(&t, g_prof[0].a, r.a);
            t0 = std::min(t0, t);
        }
        char line[256];
        for (auto& r : g_prof) {
            float st = 0.f, du = 0.f;
            cudaEventElapsedTime(&st, g_prof[0].a, r.a);
            cudaEventElapsedTime(&du, r.a, r.b);
            size_t k = 0;
            for (; k < streams.size(); ++k)
                if (streams[k] == r.s) break;
            if (k == streams.size()) streams.push_back(r.s);
            snprintf(line, sizeof(line), "%s %zu %.2f %.2f\n", r.name, k, (st - t0) * 1e3, du * 1e3);
            out += line;
        }
    }
    if (buf && buflen) {
        size_t n = out.size() < buflen - 1 ? out.size() : buflen - 1;
        memcpy(buf, out.data(), n);
        buf[n] = 0;
    }
    return GSB_OK;
}

gsb_status gsb_profile_dump(char* buf, size_t buflen) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    GSB_CUDA(cudaDeviceSynchronize());
    std::vector<std::string> names;
    std::vector<int64_t> cnt;
    std::vector<double> ms;
    for (auto& r : g_prof) {
        float t = 0.f;
        cudaEventElapsedTime(&t, r.a, r.b);
        size_t k = 0;
        for (; k < names.size(); ++k)
            if (names[k] == r.name) break;
        if (k == names.size()) {
            names.push_back(r.name);
            cnt.push_back(0);
            ms.push_back(0.0);
        }
        cnt[k] += 1;
        ms[k] += t;
        g_event_pool.push_back(r.a);
        g_event_pool.push_back(r.b);
    }
    g_prof.clear();
    std::string out;
    char line[256];
    for (size_t k = 0; k < names.size(); ++k) {
        snprintf(line, sizeof(line), "%s %lld %.6f\n", names[k].c_str(), (long long)cnt[k], ms[k]);
        out += line;
    }
    if (buf && buflen) {
        size_t n = out.size() < buflen - 1 ? out.size() : buflen - 1;
        memcpy(buf, out.data(), n);
        buf[n] = 0;
    }
    return GSB_OK;
}

gsb_status gsb_graph_create(int32_t T, const int64_t* counts, int32_t R, const int32_t* etype_src,
                            const int32_t* etype_dst, gsb_graph_t* out) {
    GSB_CHECK_ARG(out && counts && etype_src && etype_dst, "null argument");
    GSB_CHECK_ARG(T >= 1 && T <= kMaxT, "num_ntypes %d out of [1, %d]", T, kMaxT);
    GSB_CHECK_ARG(R >= 1 && R <= kMaxR, "num_etypes %d out of [1, %d]", R, kMaxR);
    Graph* G = new Graph();
    memset(&G->dev, 0, sizeof(GraphDev));
    G->dev.T = T;
    G->dev.R = R;
    G->dev.node_off[0] = 0;
    for (int t = 0; t < T; ++t) {
        if (counts[t] < 0 || counts[t] > (int64_t)INT32_MAX) {
            delete G;
            set_error("ntype %d count %lld out of range", t, (long long)counts[t]);
            return GSB_EINVAL;
        }
        G->counts[t] = counts[t];
        G->dev.node_off[t + 1] = G->dev.node_off[t] + counts[t];
    }
    for (int t = T + 1; t <= kMaxT; ++t) G->dev.node_off[t] = G->dev.node_off[T];
    G->total_nodes = G->dev.node_off[T];
    int S = 0;
    for (int r = 0; r < R; ++r) {
        if (etype_src[r] < 0 || etype_src[r] >= T || etype_dst[r] < 0 || etype_dst[r] >= T) {
            delete G;
            set_error("etype %d endpoint type out of range", r);
            return GSB_EINVAL;
        }
        G->dev.src_t[r] = etype_src[r];
        G->dev.dst_t[r] = etype_dst[r];
        int t = etype_dst[r];
        if (G->dev.n_slots[t] >= kMaxS) {
            delete G;
            set_error("ntype %d has more than %d in-relations", t, kMaxS);
            return GSB_EINVAL;
        }
        G->dev.slot_etype[t][G->dev.n_slots[t]++] = r;
    }
    for (int t = 0; t < T; ++t) S = S > G->dev.n_slots[t] ? S : G->dev.n_slots[t];
    G->dev.S = S;
    *out = reinterpret_cast<gsb_graph_t>(G);
    return GSB_OK;
}

gsb_status gsb_graph_destroy(gsb_graph_t g) {
    Graph* G = reinterpret_cast<Graph*>(g);
    if (G) delete G->cpeers_host;
    delete G;
    return GSB_OK;
}

gsb_status gsb_slot_etype(gsb_graph_t g, int32_t t, int32_t s, int32_t* etype) {
    Graph* G = reinterpret_cast<Graph*>(g);
    GSB_CHECK_ARG(G && etype && t >= 0 && t < G->dev.T, "bad argument");
    *etype = (s >= 0 && s < G->dev.n_slots[t]) ? G->dev.slot_etype[t][s] : -1;
    return GSB_OK;
}

static size_t csc_cub_bytes(int64_t n) {
    size_t b = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, b, (const uint64_t*)nullptr, (uint64_t*)nullptr, (int64_t)n, 0, 64);
    return b;
}

gsb_status gsb_csc_build_bytes(gsb_graph_t g, int32_t etype, int64_t n_edges, size_t* bytes) {
    Graph* G = reinterpret_cast<Graph*>(g);
    GSB_CHECK_ARG(G && bytes && etype >= 0 && etype < G->dev.R && n_edges >= 0, "bad argument");
    *bytes = align_up(2 * sizeof(unsigned long long)) + 2 * align_up(sizeof(uint64_t) * (size_t)(n_edges + 1)) +
             align_up(csc_cub_bytes(n_edges));
    return GSB_OK;
}

gsb_status gsb_csc_build(gsb_graph_t g, int32_t etype, const int32_t* src, const int32_t* dst, const uint8_t* keep,
                         int64_t n_edges, int64_t* indptr, int32_t* indices, int64_t* n_kept, void* ws,
                         size_t ws_bytes, void* stream) {
    Graph* G = reinterpret_cast<Graph*>(g);
    GSB_CHECK_ARG(G && etype >= 0 && etype < G->dev.R, "bad graph/etype");
    int64_t before = 0;
    return gsb_csc_build_range(g, etype, src, dst, keep, n_edges, 0, G->counts[G->dev.dst_t[etype]], indptr, indices,
                               n_kept, &before, ws, ws_bytes, stream);
}

gsb_status gsb_csc_build_range(gsb_graph_t g, int32_t etype, const int32_t* src, const int32_t* dst,
                               const uint8_t* keep, int64_t n_edges, int64_t dst_lo, int64_t dst_hi, int64_t* indptr,
                               int32_t* indices, int64_t* n_kept, int64_t* n_before, void* ws, size_t ws_bytes,
                               void* stream) {
    Graph* G = reinterpret_cast<Graph*>(g);
    GSB_CHECK_ARG(G && etype >= 0 && etype < G->dev.R, "bad graph/etype");
    GSB_CHECK_ARG(n_edges == 0 || (src && dst), "null COO");
    GSB_CHECK_ARG(indptr && indices && n_kept && n_before && ws, "null output/workspace");
    GSB_CHECK_ARG(dst_lo >= 0 && dst_lo <= dst_hi && dst_hi <= G->counts[G->dev.dst_t[etype]], "bad dst range");
    size_t need = 0;
    gsb_csc_build_bytes(g, etype, n_edges, &need);
    if (ws_bytes < need) {
        set_error("csc workspace %zu < %zu", ws_bytes, need);
        return GSB_EWORKSPACE;
    }
    cudaStream_t s = (cudaStream_t)stream;
    char* p = (char*)ws;
    unsigned long long* d_cnt = (unsigned long long*)p;
    p += align_up(2 * sizeof(unsigned long long));
    uint64_t* k_in = (uint64_t*)p;
    p += align_up(sizeof(uint64_t) * (size_t)(n_edges + 1));
    uint64_t* k_out = (uint64_t*)p;
    p += align_up(sizeof(uint64_t) * (size_t)(n_edges + 1));
    size_t cub_b = csc_cub_bytes(n_edges);
    const int64_t n_dst = dst_hi - dst_lo;
    GSB_CUDA(cudaMemsetAsync(d_cnt, 0, 2 * sizeof(unsigned long long), s));
    if (n_edges > 0) {
        GSB_LAUNCH("csc_keys", csc_keys_kernel, grid_for(n_edges, 256, kNumSMs * 32), 256, 0, s, src, dst, keep,
                   n_edges, dst_lo, dst_hi, k_in, d_cnt);
        int end_bit = 32;
        while (end_bit < 64 && ((int64_t)1 << (end_bit - 32)) <= n_dst) ++end_bit;
        GSB_CUDA(cub::DeviceRadixSort::SortKeys(p, cub_b, k_in, k_out, (int64_t)n_edges, 0, end_bit, s));
        count_launch(2 * ((end_bit + 7) / 8));
    }
    GSB_LAUNCH("csc_finish", csc_finish_kernel, grid_for(n_edges > n_dst ? n_edges : n_dst + 1, 256, kNumSMs * 32),
               256, 0, s, k_out, d_cnt, n_dst, indptr, indices);
    unsigned long long h[2] = {0, 0};
    GSB_CUDA(cudaMemcpyAsync(h, d_cnt, sizeof(h), cudaMemcpyDeviceToHost, s));
    GSB_CUDA(cudaStreamSynchronize(s));
    *n_kept = (int64_t)h[0];
    *n_before = (int64_t)h[1];
    G->dev.indptr[etype] = indptr;
    G->dev.indices[etype] = indices;
    G->dev.eid_base[etype] = (int64_t)h[1];
    G->n_edges[etype] = (int64_t)h[0];
    return GSB_OK;
}

gsb_status gsb_graph_set_csc(gsb_graph_t g, int32_t etype, const int64_t* indptr, const int32_t* indices,
                             int64_t n_edges, int64_t eid_base) {
    Graph* G = reinterpret_cast<Graph*>(g);
    GSB_CHECK_ARG(G && etype >= 0 && etype < G->dev.R && indptr && (indices || n_edges == 0), "bad argument");
    G->dev.indptr[etype] = indptr;
    G->dev.indices[etype] = indices;
    G->dev.eid_base[etype] = eid_base;
    G->n_edges[etype] = n_edges;
    return GSB_OK;
}

gsb_status gsb_graph_set_features(gsb_graph_t g, int32_t ntype, const void* feat, int32_t dim, int32_t dtype) {
    Graph* G = reinterpret_cast<Graph*>(g);
    GSB_CHECK_ARG(G && ntype >= 0 && ntype < G->dev.T && feat, "bad argument");
    GSB_CHECK_ARG(((uintptr_t)feat & 15) == 0, "feature table must be 16-byte aligned");
    gsb_status st = set_feature_format(G, ntype, dim, dtype);
    if (st != GSB_OK) return st;
    G->dev.feat[ntype] = static_cast<const char*>(feat);
    return GSB_OK;
}

gsb_status gsb_gather(gsb_graph_t g, const int64_t* gid, int64_t n, void* out, void* stream) {
    Graph* G = reinterpret_cast<Graph*>(g);
    GSB_CHECK_ARG(G && (n == 0 || (gid && out)), "bad argument");
    for (int t = 0; t < G->dev.T; ++t) GSB_CHECK_ARG(G->dev.feat[t], "features of ntype %d not registered", t);
    GSB_CHECK_ARG(G->dev.feat_dim > 0, "gather needs one feature width for all ntypes");
    if (n == 0) return GSB_OK;
    return launch_gather(G, gid, nullptr, n, n, out, (cudaStream_t)stream);
}

gsb_status gsb_adam_step(float* p, const float* g, float* m, float* v, int64_t n, float lr, float b1, float b2,
                         float eps, int32_t t, const int32_t* t_dev, void* stream) {
    GSB_CHECK_ARG(p && g && m && v && n >= 0 && (t >= 1 || t_dev), "bad argument");
    if (t < 1) t = 1;
    if (n == 0) return GSB_OK;
    float c1 = 1.f - powf(b1, (float)t);
    float c2 = 1.f - powf(b2, (float)t);
    GSB_CHECK_ARG(((uintptr_t)p & 15) == 0 && ((uintptr_t)g & 15) == 0 && ((uintptr_t)m & 15) == 0 &&
                      ((uintptr_t)v & 15) == 0, "adam buffers must be 16-byte aligned");
    GSB_LAUNCH("adam", adam_kernel, grid_for((n + 3) / 4, 256, kNumSMs * 4), 256, 0, (cudaStream_t)stream, p, g, m, v, n, lr,
               b1, b2, eps, c1, c2, t_dev, (float*)nullptr, (float*)nullptr, AdamPad{0, 0, 0, 0, nullptr, nullptr});
    return GSB_OK;
}

gsb_status gsb_adam_step_split(float* p, const float* g, float* m, float* v, int64_t n, float lr, float b1, float b2,
                               float eps, int32_t t, const int32_t* t_dev, float* hi, float* lo, int64_t pad_off,
                               int32_t pad_rows, int32_t pad_cols, int32_t pad_ld, float* pad_hi, float* pad_lo,
                               void* stream) {
    GSB_CHECK_ARG(p && g && m && v && hi && lo && n >= 0 && (t >= 1 || t_dev), "bad argument");
    GSB_CHECK_ARG(!pad_hi || (pad_lo && pad_off >= 0 && pad_rows >= 1 && pad_cols >= 1 && pad_ld >= pad_cols &&
                              pad_off + (int64_t)pad_rows * pad_cols <= n),
                  "bad padded segment");
    if (t < 1) t = 1;
    if (n == 0) return GSB_OK;
    float c1 = 1.f - powf(b1, (float)t);
    float c2 = 1.f - powf(b2, (float)t);
    GSB_CHECK_ARG(((uintptr_t)p & 15) == 0 && ((uintptr_t)g & 15) == 0 && ((uintptr_t)m & 15) == 0 &&
                      ((uintptr_t)v & 15) == 0 && ((uintptr_t)hi & 15) == 0 && ((uintptr_t)lo & 15) == 0,
                  "adam buffers must be 16-byte aligned");
    GSB_LAUNCH("adam", adam_kernel, grid_for((n + 3) / 4, 256, kNumSMs * 4), 256, 0, (cudaStream_t)stream, p, g, m, v, n, lr,
               b1, b2, eps, c1, c2, t_dev, hi, lo, AdamPad{pad_off, pad_rows, pad_cols, pad_ld, pad_hi, pad_lo});
    return GSB_OK;
}

gsb_status gsb_counter_add(int32_t* counter, int32_t delta, void* stream) {
    GSB_CHECK_ARG(counter, "null counter");
    GSB_LAUNCH("counter_add", counter_add_kernel, 1, 1, 0, (cudaStream_t)stream, counter, delta);
    return GSB_OK;
}

gsb_status gsb_spin(int64_t ns, void* stream) {
    GSB_LAUNCH("spin", spin_kernel, 1, 32, 0, (cudaStream_t)stream, ns);
    return GSB_OK;
}

}  // extern "C"
