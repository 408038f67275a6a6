// weights.cu -- tf32 hi / lo images of the layer weights for the TMA-everything GEMM
// (gemm_tma3.cuh).  3xTF32 needs every fp32 operand split into hi and lo; a weight is the B
// operand of every CTA of a GEMM, so instead of each CTA splitting the same W in shared memory,
// W is split once per step (hi = rna_tf32(W), lo = rna_tf32(W - hi), in W's own layout) into
// caller-owned images that the NN / NT GEMMs TMA straight into the MMA stage.
// Contract: include/gsb.h "Weight images".
#include <mutex>

#include "gemm_tma.cuh"
#include "gsb_internal.cuh"

namespace gsb {

static std::mutex g_wi_mu;
static std::vector<WeightImage> g_wi;

const WeightImage* find_weight_image(const float* W) {
    std::lock_guard<std::mutex> lk(g_wi_mu);
    for (const WeightImage& w : g_wi)
        if (w.W == W) return &w;
    return nullptr;
}

static size_t wi_floats(int slots, int K, int N, int ldn) {
    (void)N;
    return 2 * (size_t)slots * K * ldn;
}

constexpr int kMaxImages = 8;
struct WiBatch {
    int n;
    WeightImage w[kMaxImages];
};

// one thread per weight element of every registered image: split into hi / lo (W layout, ldn)
__global__ void __launch_bounds__(256) weight_split_kernel(WiBatch b) {
    GSB_PDL_ENTRY();
    for (int q = 0; q < b.n; ++q) {
        const WeightImage& w = b.w[q];
        const uint32_t total = (uint32_t)w.slots * (uint32_t)w.K * (uint32_t)w.N;   // < 2^32 (checked)
        for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
            const uint32_t r = i / (uint32_t)w.N;       // row (slot, k)
            const int n = (int)(i - r * (uint32_t)w.N);
            uint32_t hi, lo;
            umma::split_tf32(w.W[i], hi, lo);
            const int64_t o = (int64_t)r * w.ldn + n;
            w.hi[o] = __uint_as_float(hi);
            w.lo[o] = __uint_as_float(lo);
        }
    }
}

}  // namespace gsb

using namespace gsb;

extern "C" {

gsb_status gsb_weight_images_bytes(int32_t slots, int32_t K, int32_t N, size_t* bytes) {
    GSB_CHECK_ARG(bytes && slots >= 1 && K >= 1 && N >= 1, "bad argument");
    *bytes = sizeof(float) * wi_floats(slots, K, N, (N + 3) / 4 * 4);
    return GSB_OK;
}

gsb_status gsb_weight_images_register(const float* W, int32_t slots, int32_t K, int32_t N, void* img,
                                      size_t img_bytes, void* stream) {
    GSB_CHECK_ARG(W && img && slots >= 1 && K >= 1 && N >= 1, "bad argument");
    GSB_CHECK_ARG((int64_t)slots * K * N < ((int64_t)1 << 32), "weight too large for an image");
    GSB_CHECK_ARG(((uintptr_t)img & 15) == 0, "image buffer must be 16-byte aligned");
    const int ldn = (N + 3) / 4 * 4;
    GSB_CHECK_ARG(img_bytes >= sizeof(float) * wi_floats(slots, K, N, ldn), "image buffer too small");
    WeightImage w;
    w.W = W;
    w.slots = slots;
    w.K = K;
    w.N = N;
    w.ldn = ldn;
    float* p = static_cast<float*>(img);
    w.hi = p;
    w.lo = p + (size_t)slots * K * ldn;
    // padding columns stay zero (the NT GEMM reduces over them)
    GSB_CUDA(cudaMemsetAsync(img, 0, img_bytes, (cudaStream_t)stream));
    std::lock_guard<std::mutex> lk(g_wi_mu);
    for (WeightImage& x : g_wi)
        if (x.W == W) {
            x = w;
            return GSB_OK;
        }
    GSB_CHECK_ARG(g_wi.size() < 64, "too many weight images");
    g_wi.push_back(w);
    return GSB_OK;
}

gsb_status gsb_weight_images_register_split(const float* W, int32_t slots, int32_t K, int32_t N, float* hi,
                                            float* lo) {
    GSB_CHECK_ARG(W && hi && lo && slots >= 1 && K >= 1 && N >= 1, "bad argument");
    GSB_CHECK_ARG(N % 4 == 0, "N %d must be a multiple of 4 (16-B rows)", N);
    GSB_CHECK_ARG(((uintptr_t)hi & 15) == 0 && ((uintptr_t)lo & 15) == 0, "images must be 16-byte aligned");
    WeightImage w;
    w.W = W;
    w.slots = slots;
    w.K = K;
    w.N = N;
    w.ldn = N;
    w.hi = hi;
    w.lo = lo;
    std::lock_guard<std::mutex> lk(g_wi_mu);
    for (WeightImage& x : g_wi)
        if (x.W == W) {
            x = w;
            return GSB_OK;
        }
    GSB_CHECK_ARG(g_wi.size() < 64, "too many weight images");
    g_wi.push_back(w);
    return GSB_OK;
}

gsb_status gsb_weight_images_unregister(const float* W) {
    std::lock_guard<std::mutex> lk(g_wi_mu);
    for (size_t i = 0; i < g_wi.size(); ++i)
        if (g_wi[i].W == W) {
            g_wi.erase(g_wi.begin() + (long)i);
            break;
        }
    return GSB_OK;
}

gsb_status gsb_weight_images_refresh(const float* const* Ws, int32_t n, void* stream) {
    GSB_CHECK_ARG(Ws && n >= 1 && n <= kMaxImages, "1..%d weights per refresh", kMaxImages);
    WiBatch b;
    b.n = n;
    int64_t total = 0;
    for (int q = 0; q < n; ++q) {
        const WeightImage* w = find_weight_image(Ws[q]);
        GSB_CHECK_ARG(w, "weight %d has no registered image", q);
        b.w[q] = *w;
        total = std::max<int64_t>(total, (int64_t)w->slots * w->K * w->N);
    }
    GSB_LAUNCH("weight_split", weight_split_kernel, grid_for(total, 256, kNumSMs * 4), 256, 0, (cudaStream_t)stream, b);
    return GSB_OK;
}

}  // extern "C"
