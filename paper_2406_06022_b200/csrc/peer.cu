// peer.cu -- NVLink peer access to other GPUs' feature shards (CUDA IPC).  With the shards
// registered, the fused layer-0 gather+aggregation reads every source row straight from its
// owner's HBM over NVLink/NVSwitch: the feature fetch of §8(e) happens inside the compute
// kernel (no all-to-all, no host-synced sizes, CUDA-graph capturable).
// Contract: include/gsb.h "Peer feature access".
#include <cuda.h>

#include "gsb_internal.cuh"

namespace gsb {

typedef CUresult (*PFN_getAddressRange)(CUdeviceptr*, size_t*, CUdeviceptr);

static PFN_getAddressRange address_range_fn() {
    static PFN_getAddressRange fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_getAddressRange>(p);
    }
    return fn;
}

}  // namespace gsb

using namespace gsb;

extern "C" {

gsb_status gsb_ipc_handle(const void* dev_ptr, void* handle_out, int64_t* offset_out) {
    GSB_CHECK_ARG(dev_ptr && handle_out && offset_out, "null argument");
    PFN_getAddressRange fn = address_range_fn();
    GSB_CHECK_ARG(fn, "cuMemGetAddressRange entry point unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (fn(&base, &size, (CUdeviceptr)dev_ptr) != CUDA_SUCCESS) {
        set_error("cuMemGetAddressRange failed");
        return GSB_ECUDA;
    }
    cudaIpcMemHandle_t h;
    GSB_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
    memcpy(handle_out, &h, sizeof(h));
    *offset_out = (int64_t)((CUdeviceptr)dev_ptr - base);
    return GSB_OK;
}

gsb_status gsb_ipc_open(const void* handle, int64_t offset, void** dev_ptr_out) {
    GSB_CHECK_ARG(handle && dev_ptr_out && offset >= 0, "bad argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    void* base = nullptr;
    GSB_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    *dev_ptr_out = static_cast<char*>(base) + offset;
    return GSB_OK;
}

gsb_status gsb_ipc_close(void* base_ptr) {
    GSB_CUDA(cudaIpcCloseMemHandle(base_ptr));
    return GSB_OK;
}

gsb_status gsb_graph_set_feature_peers(gsb_graph_t g, int32_t ntype, int32_t world, const int64_t* bounds,
                                       const void* const* ptrs, int32_t dim, int32_t dtype) {
    Graph* G = reinterpret_cast<Graph*>(g);
    GSB_CHECK_ARG(G && bounds && ptrs && ntype >= 0 && ntype < G->dev.T, "bad argument");
    GSB_CHECK_ARG(world >= 1 && world <= kMaxPeers, "world %d out of [1, %d]", world, kMaxPeers);
    GSB_CHECK_ARG(bounds[0] == 0 && bounds[world] == G->counts[ntype], "bounds must span [0, count)");
    gsb_status st = set_feature_format(G, ntype, dim, dtype);
    if (st != GSB_OK) return st;
    G->dev.nparts = world;
    for (int w = 0; w <= world; ++w) G->dev.plo[ntype][w] = bounds[w];
    for (int w = 0; w < world; ++w) {
        GSB_CHECK_ARG(ptrs[w] || bounds[w + 1] == bounds[w], "null shard pointer for rank %d", w);
        GSB_CHECK_ARG(((uintptr_t)ptrs[w] & 15) == 0, "shard of rank %d not 16-byte aligned", w);
        G->dev.peer[ntype][w] = static_cast<const char*>(ptrs[w]);
    }
    // the local-table pointer is unused in partitioned mode but marks the ntype as registered
    G->dev.feat[ntype] = ptrs[0] ? static_cast<const char*>(ptrs[0]) : reinterpret_cast<const char*>(16);
    return GSB_OK;
}

gsb_status gsb_csc_peers_bytes(size_t* bytes) {
    GSB_CHECK_ARG(bytes, "null argument");
    *bytes = sizeof(CscPeers);
    return GSB_OK;
}

gsb_status gsb_graph_set_csc_peers(gsb_graph_t g, void* table_dev, int32_t etype, int32_t world,
                                   const int64_t* bounds, const int64_t* const* indptr_w,
                                   const int32_t* const* indices_w, const int64_t* eid_base_w, int64_t n_edges_total,
                                   void* stream) {
    Graph* G = reinterpret_cast<Graph*>(g);
    GSB_CHECK_ARG(G && table_dev && bounds && indptr_w && indices_w && eid_base_w, "null argument");
    GSB_CHECK_ARG(etype >= 0 && etype < G->dev.R, "etype %d out of range", etype);
    GSB_CHECK_ARG(world >= 1 && world <= kMaxPeers, "world %d out of [1, %d]", world, kMaxPeers);
    GSB_CHECK_ARG(((uintptr_t)table_dev & 15) == 0, "table must be 16-byte aligned");
    if (!G->cpeers_host) {
        G->cpeers_host = new CscPeers();
        memset(G->cpeers_host, 0, sizeof(CscPeers));
    }
    CscPeers& P = *G->cpeers_host;
    GSB_CHECK_ARG(P.world == 0 || P.world == world, "world changed between etypes");
    P.world = world;
    for (int t = 0; t < G->dev.T; ++t) {
        GSB_CHECK_ARG(bounds[t * (world + 1)] == 0 && bounds[t * (world + 1) + world] == G->counts[t],
                      "bounds of ntype %d must span [0, count)", t);
        for (int w = 0; w <= world; ++w) P.lo[t][w] = bounds[t * (world + 1) + w];
    }
    for (int w = 0; w < world; ++w) {
        GSB_CHECK_ARG(indptr_w[w], "null indptr of rank %d", w);
        P.indptr[etype][w] = indptr_w[w];
        P.indices[etype][w] = indices_w[w];
        P.eid_base[etype][w] = eid_base_w[w];
    }
    GSB_CHECK_ARG(n_edges_total >= 0, "bad n_edges_total");
    // capacities (fanout ALL, full-graph sweeps) are sized by the whole graph's edge count
    G->n_edges[etype] = n_edges_total;
    cudaStream_t s = (cudaStream_t)stream;
    GSB_CUDA(cudaMemcpyAsync(table_dev, &P, sizeof(CscPeers), cudaMemcpyHostToDevice, s));
    GSB_CUDA(cudaStreamSynchronize(s));
    G->dev.cpeers = static_cast<const CscPeers*>(table_dev);
    return GSB_OK;
}

}  // extern "C"
