// probe_green.cu -- can the two pipeline phases be given disjoint SM sets with green contexts?
// Splits the SMs into two green contexts, creates a stream in each, and checks (via %smid)
// that kernels launched with the runtime API -- directly and from a CUDA graph captured on
// the green stream -- stay inside their partition, with memory from cudaMalloc (primary ctx).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 scripts/probe_green.cu -o scripts/probe_green.bin -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdio.h>

#include <set>
#include <vector>

#define CU(x)                                                               \
    do {                                                                    \
        CUresult r = (x);                                                   \
        if (r != CUDA_SUCCESS) {                                            \
            const char* m = nullptr;                                        \
            cuGetErrorString(r, &m);                                        \
            printf("%s:%d %s -> %d %s\n", __FILE__, __LINE__, #x, (int)r, m); \
            return 1;                                                       \
        }                                                                   \
    } while (0)
#define CK(x)                                                                          \
    do {                                                                               \
        cudaError_t e = (x);                                                           \
        if (e != cudaSuccess) {                                                        \
            printf("%s:%d %s -> %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
            return 1;                                                                  \
        }                                                                              \
    } while (0)

__global__ void smid_kernel(int* out, long long spin) {
    unsigned s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    if (threadIdx.x == 0) out[blockIdx.x] = (int)s;
    long long t0 = clock64();
    while (clock64() - t0 < spin) {
    }
}

static std::set<int> sms(const std::vector<int>& v) { return std::set<int>(v.begin(), v.end()); }

int main() {
    CK(cudaFree(0));
    CUdevice dev;
    CU(cuDeviceGet(&dev, 0));
    CUdevResource all;
    CU(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
    printf("device SMs %u\n", all.sm.smCount);
    CUdevResource part[1], rest;
    unsigned n = 1;
    CU(cuDevSmResourceSplitByCount(part, &n, &all, &rest, 0, 40));
    printf("split: group %u SMs, remainder %u SMs\n", part[0].sm.smCount, rest.sm.smCount);
    CUdevResourceDesc dA, dB;
    CU(cuDevResourceGenerateDesc(&dA, part, 1));
    CU(cuDevResourceGenerateDesc(&dB, &rest, 1));
    CUgreenCtx gA, gB;
    CU(cuGreenCtxCreate(&gA, dA, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CU(cuGreenCtxCreate(&gB, dB, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream sA, sB;
    CU(cuGreenCtxStreamCreate(&sA, gA, CU_STREAM_NON_BLOCKING, 0));
    CU(cuGreenCtxStreamCreate(&sB, gB, CU_STREAM_NON_BLOCKING, 0));
    const int nb = 1024;
    int *bA, *bB;
    CK(cudaMalloc(&bA, nb * 4));
    CK(cudaMalloc(&bB, nb * 4));
    // direct launches on both streams at once
    smid_kernel<<<nb, 128, 0, (cudaStream_t)sA>>>(bA, 200000);
    smid_kernel<<<nb, 128, 0, (cudaStream_t)sB>>>(bB, 200000);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<int> hA(nb), hB(nb);
    CK(cudaMemcpy(hA.data(), bA, nb * 4, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hB.data(), bB, nb * 4, cudaMemcpyDeviceToHost));
    auto a = sms(hA), b = sms(hB);
    int both = 0;
    for (int x : a) both += b.count(x);
    printf("direct: stream A used %zu SMs, stream B %zu SMs, shared %d\n", a.size(), b.size(), both);
    // graph captured on the green stream A, replayed on A
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture((cudaStream_t)sA, cudaStreamCaptureModeGlobal));
    smid_kernel<<<nb, 128, 0, (cudaStream_t)sA>>>(bA, 100000);
    CK(cudaStreamEndCapture((cudaStream_t)sA, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    CK(cudaMemset(bA, 0xff, nb * 4));
    CK(cudaGraphLaunch(ge, (cudaStream_t)sA));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(hA.data(), bA, nb * 4, cudaMemcpyDeviceToHost));
    auto ga = sms(hA);
    both = 0;
    for (int x : ga) both += a.count(x);
    printf("graph on A: used %zu SMs, %d of them in A's direct set\n", ga.size(), both);
    // the same graph launched on an ordinary stream of the primary context
    cudaStream_t sp;
    CK(cudaStreamCreateWithFlags(&sp, cudaStreamNonBlocking));
    CK(cudaGraphLaunch(ge, sp));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(hA.data(), bA, nb * 4, cudaMemcpyDeviceToHost));
    auto gp = sms(hA);
    printf("graph captured on A, launched on a primary-ctx stream: used %zu SMs\n", gp.size());
    return 0;
}
