/*
 * gsb.h -- C ABI of libgsb: a B200-native (sm_100a) RGCN mini-batch training step,
 * after GraphStorm (Zheng et al., arXiv 2406.06022, KDD'24).
 *
 * Citations: "P:Lnnn" = /root/reference/PAPER.md line nnn; "S:Lnnn" = SPEC.md line nnn;
 * "R-x" = a reading of a silent / garbled passage, listed in DESIGN.md §Readings.
 *
 * Conventions (all entry points):
 *  - Plain C types only.  "device" pointers are CUDA global-memory pointers (e.g. a
 *    torch tensor's data_ptr); "host" pointers are CPU memory.  `stream` is a
 *    cudaStream_t passed as void* (NULL = legacy default stream).
 *  - Ownership: the library never allocates device memory.  Every device buffer is
 *    caller-owned; sizes come from the *_bytes / *_floats queries.  Handles
 *    (gsb_graph_t, gsb_blocks_t) are small host structs owned by the library, freed by
 *    their *_destroy call; they keep (do not copy) the device pointers registered in them.
 *  - Asynchrony: every call only enqueues work on `stream` and returns, except the
 *    calls documented as "syncs".  No call performs a host<->device transfer of data
 *    sizes on the hot path, so a whole train step can be captured in a CUDA graph.
 *  - Errors: argument / shape / capacity errors return a non-zero gsb_status
 *    synchronously and set gsb_last_error() (thread-local text).  Errors detected by a
 *    kernel (unknown node id, frontier not grouped by node type, capacity overflow) are
 *    latched in a device word inside the arena and returned by gsb_blocks_poll_error().
 *  - Layouts: node features are row-major [rows][dim] fp32 or bf16 (GSB_F32 / GSB_BF16,
 *    one format for all node types; bf16 values are widened exactly to fp32 when read);
 *    hidden states, activations and parameters are row-major fp32.  Global node
 *    ids (gid) are type-major: gid = node_off[t] + local id (R-gid).  Relation weights W
 *    of a layer are row-major [R+1][d_in][d_out]; slot R is W_self.
 *  - Threads: calls on one handle are not thread-safe; separate handles are independent.
 */
#ifndef GSB_H_
#define GSB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t gsb_status;
#define GSB_OK 0
#define GSB_EINVAL 1      /* bad argument / shape / unsupported configuration        */
#define GSB_EWORKSPACE 2  /* caller-provided buffer too small                         */
#define GSB_ECUDA 3       /* a CUDA runtime call or kernel launch failed              */
#define GSB_EDEVICE 4     /* a latched device-side error (see gsb_blocks_poll_error)  */
#define GSB_ECALLBACK 5   /* a host callback (gsb_exchange_fn) reported failure         */

/* feature element types */
#define GSB_F32 0
#define GSB_BF16 1

#define GSB_MAX_NTYPES 8
#define GSB_MAX_ETYPES 32
#define GSB_MAX_SLOTS 8    /* max in-relations of one node type */
#define GSB_MAX_LAYERS 4
#define GSB_MAX_FANOUT 32  /* Floyd draws are resolved by one warp; -1 (ALL) is unbounded */

/* Thread-local message for the last non-OK status of this thread. */
const char* gsb_last_error(void);
/* ABI version (major*100 + minor). */
int32_t gsb_version(void);

/* --------------------------------------------------------------------------------------
 * Instrumentation (used by bench.py for the roofline numbers; off by default).
 *  gsb_launch_count: number of kernels this library has launched since load.
 *  gsb_profile_enable(1): from now on every launch is bracketed by CUDA events on its
 *    own stream.  gsb_profile_dump (syncs the device) writes one line per kernel name,
 *    "name launches total_ms\n", into buf (truncated to buflen) and clears the records.
 * ------------------------------------------------------------------------------------ */
int64_t gsb_launch_count(void);
gsb_status gsb_profile_enable(int32_t on);
gsb_status gsb_profile_dump(char* buf, size_t buflen);
/* Tools: one line per launch profiled since the last dump, in enqueue order -- "name stream
 * start_us dur_us" (stream = index in order of first use, start relative to the earliest
 * launch); does not clear the records (gsb_profile_dump does). */
gsb_status gsb_profile_timeline(char* buf, size_t buflen);

/* ======================================================================================
 * Graph store ("distributed graph engine"; S:L225 load_partition, S:L240 edge
 * owned by its destination).  One CSC per etype over destination nodes of its dst type:
 *   indptr  int64 [n_dst + 1]   (device)
 *   indices int32 [n_edges]     (device) src local id, ascending within a segment (R-csc)
 *   eid of an edge = eid_base[etype] + its CSC position (R-eid; no array stored).
 * ==================================================================================== */
typedef struct gsb_graph* gsb_graph_t;

/* Create the (host) schema handle.  ntype_count: host [num_ntypes] node counts;
 * etype_src / etype_dst: host [num_etypes] node type ids.  Fails with GSB_EINVAL for
 * num_ntypes > GSB_MAX_NTYPES, num_etypes > GSB_MAX_ETYPES, more than GSB_MAX_SLOTS
 * etypes into one node type, or > 2^31 nodes in one type. */
gsb_status gsb_graph_create(int32_t num_ntypes, const int64_t* ntype_count, int32_t num_etypes,
                            const int32_t* etype_src, const int32_t* etype_dst, gsb_graph_t* out);
gsb_status gsb_graph_destroy(gsb_graph_t g);

/* Device workspace bytes needed by gsb_csc_build for n_edges COO edges of `etype`. */
gsb_status gsb_csc_build_bytes(gsb_graph_t g, int32_t etype, int64_t n_edges, size_t* bytes);

/* Build the CSC of `etype` on the device from a COO edge list (src, dst: device int32
 * local ids, n_edges).  keep: optional device uint8 mask (NULL = keep all); val/test LP
 * edges are dropped this way.  Output: indptr (device int64 [n_dst+1]), indices
 * (device int32, capacity n_edges).  *n_kept (host) receives the kept edge count.
 * Registers indptr/indices in g for `etype` (eid_base 0).  Syncs `stream`. */
gsb_status gsb_csc_build(gsb_graph_t g, int32_t etype, const int32_t* src, const int32_t* dst,
                         const uint8_t* keep, int64_t n_edges, int64_t* indptr, int32_t* indices,
                         int64_t* n_kept, void* ws, size_t ws_bytes, void* stream);

/* Partitioned build (§8(e): the graph partitioned by node ID, edges owned by their dst's
 * owner): as gsb_csc_build over the kept edges whose dst local id lies in
 * [dst_lo, dst_hi) only, with dst ids shifted by -dst_lo (indptr: device int64
 * [dst_hi - dst_lo + 1]).  *n_before (host) receives the kept edges with dst < dst_lo: the
 * global CSC position of this range's first edge, registered as the etype's eid_base (edge ids
 * stay those of the whole graph, R-eid).  gsb_csc_build = the range [0, count). */
gsb_status gsb_csc_build_range(gsb_graph_t g, int32_t etype, const int32_t* src, const int32_t* dst,
                               const uint8_t* keep, int64_t n_edges, int64_t dst_lo, int64_t dst_hi, int64_t* indptr,
                               int32_t* indices, int64_t* n_kept, int64_t* n_before, void* ws, size_t ws_bytes,
                               void* stream);

/* Register a prebuilt CSC (device pointers) for `etype`; eid_base is added to CSC
 * positions to form edge ids (multi-GPU partitions). */
gsb_status gsb_graph_set_csc(gsb_graph_t g, int32_t etype, const int64_t* indptr, const int32_t* indices,
                             int64_t n_edges, int64_t eid_base);

/* Register the feature table of `ntype`: device [ntype_count][dim] row-major, element type
 * dtype (GSB_F32 / GSB_BF16), 16-byte aligned, dim * element size a multiple of 16
 * (P:L86 distributed tensors).  All ntypes share one dtype; widths may differ per ntype
 * (input-encoder graphs), but the fused layer-0 path and the gathers need one width. */
gsb_status gsb_graph_set_features(gsb_graph_t g, int32_t ntype, const void* feat, int32_t dim, int32_t dtype);

/* Feature gather by global id (§8(a) a5; S:L299 fetch_features):
 *   out[i, :] = F_{t(i)}[gid[i] - node_off[t(i)], :]   for i < n   (exact copy)
 * gid: device int64 [n]; out: device [n][dim] in the feature dtype.  A gid outside
 * [0, total nodes) yields a zero row. */
gsb_status gsb_gather(gsb_graph_t g, const int64_t* gid, int64_t n, void* out, void* stream);

/* ======================================================================================
 * Mini-batch sampling into message-flow blocks (P:L58, P:L86 on-the-fly sampling;
 * Fig. 4 P:L122-128 fanout/batch; Fig. 8 P:L480-486 blocks[i]).
 *
 * gsb_sample draws L hops from the seeds.  Hop h (1-based from the seeds) uses fanout
 * f[L-h] (layer l consumes the block of hop L-l; blocks[0] is the input layer, R-fanout).
 * For every frontier node v and every etype r into type(v) (ascending r) it keeps
 * min(f, deg'_r(v)) in-edges chosen uniformly without replacement (R-wor) by Floyd's
 * algorithm on Philox4x32-10 draws keyed by (rng_seed; dst gid, etype, hop, draw, step)
 * (R-rng, R-floyd); f = -1 keeps all.  deg' excludes the batch's LP target edges
 * (u,v) in excl_etype and (v,u) in excl_rev_etype (R-excl).
 * Relabel (R-relabel): per ntype, src list = [frontier nodes of that type, frontier order]
 * ++ ascending unique new sampled sources; the next frontier is their concatenation.
 * Frontier / seeds must be grouped by node type in ascending type order (latched error
 * otherwise).  All sizes after the seeds stay on the device.
 * ==================================================================================== */
typedef struct gsb_blocks* gsb_blocks_t;

/* fanouts: host [num_layers], f[l] for layer l, each -1 or 1..GSB_MAX_FANOUT.
 * max_seeds: capacity of the seed frontier; max_excl: capacity of LP exclusion pairs. */
/* Host callback of the NCCL frontier exchange (gsb_blocks_set_exchange).  phase 0: the library
 * has bucketed this hop's frontier by owner (send_cnt, req_send); the callback runs the
 * all-to-alls of the counts and of the request ids into req_recv (grouped by source rank) on
 * `stream` and stores the received counts per rank in counts[0..world).  phase 1: the library
 * has sampled the received requests (srv_cnt per (request, slot), srv_gid / srv_eid edges,
 * srv_wcnt edges per requesting rank); the callback returns them with all-to-alls into
 * resp_cnt (this rank's requests, in req_send order) and resp_gid / resp_eid.  Returns 0 on
 * success. */
typedef int32_t (*gsb_exchange_fn)(void* user, int32_t phase, int32_t hop, void* stream, int64_t* counts);

/* Caller-owned device buffers of the exchange (sizes from gsb_exchange_sizes):
 * int64 req_send[cap_dst], int32 req_perm[cap_dst], int64 send_cnt[world], cursor[world],
 * int64 req_recv[cap_recv], int64 xoff[world+1], srv_meta[meta_bytes],
 * int64 srv_cnt[srv_cnt_len], srv_seg[cap_recv*S+1], srv_gid / srv_eid[cap_srv_e],
 * int64 srv_wcnt[world], resp_cnt / resp_seg[cap_dst*S+1], resp_gid / resp_eid[cap_resp_e]. */
typedef struct {
    int64_t* req_send; int32_t* req_perm; int64_t* send_cnt; int64_t* cursor;
    int64_t* req_recv; int64_t cap_recv; int64_t* xoff; void* srv_meta;
    int64_t* srv_cnt; int64_t* srv_seg; int64_t* srv_gid; int64_t* srv_eid; int64_t cap_srv_e; int64_t* srv_wcnt;
    int64_t* resp_cnt; int64_t* resp_seg; int64_t* resp_gid; int64_t* resp_eid; int64_t cap_resp_e;
} gsb_exchange_bufs;

gsb_status gsb_blocks_create(gsb_graph_t g, int32_t num_layers, const int32_t* fanouts, int64_t max_seeds,
                             int64_t max_excl, gsb_blocks_t* out);
gsb_status gsb_blocks_destroy(gsb_blocks_t b);
/* NCCL frontier exchange (§8(e) C2/C3; P:L86 sampling on a distributed graph, P:L172 remote
 * partition access): with first_hop > 0, hops >= first_hop of gsb_sample send every frontier
 * node to its owner (bounds of gsb_graph_set_csc_peers: this rank's own CSC shard is the only
 * one it reads), the owners sample the requests with the keyed RNG (requester's step word:
 * this rank's + requester - rank) and reply with the counts and edges; the blocks are those of
 * a whole-graph sampler, bit-exact.  fn runs the all-to-alls (see gsb_exchange_fn);
 * gsb_sample then synchronizes the host twice per exchanged hop.  first_hop 0 turns it off. */
gsb_status gsb_blocks_set_exchange(gsb_blocks_t b, int32_t world, int32_t rank, int32_t first_hop,
                                   const gsb_exchange_bufs* bufs, gsb_exchange_fn fn, void* user);
gsb_status gsb_exchange_sizes(gsb_blocks_t b, int32_t world, int64_t* cap_dst, int64_t* cap_recv,
                              int64_t* cap_srv_e, int64_t* cap_resp_e, int64_t* srv_cnt_len, int64_t* meta_bytes);

/* Device arena bytes for all blocks of one mini-batch (upper bounds). */
gsb_status gsb_blocks_arena_bytes(gsb_blocks_t b, size_t* bytes);
/* One-time arena initialisation (node maps to "absent").  Must precede the first sample. */
gsb_status gsb_blocks_init_arena(gsb_blocks_t b, void* arena, size_t arena_bytes, void* stream);

/* Arguments of one gsb_sample call.
 *  seeds      device int64 gids; distinct, grouped by ntype in ascending type order
 *  n_seeds    host count (or, when n_seeds_dev != NULL, the capacity bound <= max_seeds)
 *  n_seeds_dev  optional device int64 count (e.g. written by gsb_lp_seeds)
 *  rng_seed   Philox key; step: counter word (R-rng); step_dev: optional device uint32
 *             overriding `step` (lets a captured CUDA graph advance the step on device)
 *  excl_u/excl_v  optional device int64 gids [n_excl] of LP batch positives (u,v) of
 *             excl_etype; their reverses are excluded from excl_rev_etype (-1 = none). */
typedef struct {
    const int64_t* seeds;
    int64_t n_seeds;
    const int64_t* n_seeds_dev;
    uint64_t rng_seed;
    uint32_t step;
    const uint32_t* step_dev;
    const int64_t* excl_u;
    const int64_t* excl_v;
    int64_t n_excl;
    int32_t excl_etype;
    int32_t excl_rev_etype;
} gsb_sample_args;

/* Samples all hops of one mini-batch into the arena. */
gsb_status gsb_sample(gsb_blocks_t b, const gsb_sample_args* args, void* arena, size_t arena_bytes, void* stream);

/* Sizes of the block of `layer` (syncs `stream`): n_dst, n_src, n_edges and the
 * per-ntype dst / src row counts (host arrays [num_ntypes]). */
gsb_status gsb_block_sizes(gsb_blocks_t b, const void* arena, int32_t layer, int64_t* n_dst, int64_t* n_src,
                           int64_t* n_edges, int64_t* dst_type_cnt, int64_t* src_type_cnt, void* stream);

/* Device views of the block of `layer` (pointers into the arena).  Layout:
 *   dst_gid  int64 [n_dst]          frontier (= src rows [0..] of the same type, dst prefix)
 *   src_gid  int64 [n_src]          next frontier, type-grouped
 *   seg_ptr  int64 [n_dst*S+1]      edge offsets of segment (dst row j, slot s), S = slots;
 *                                   slot s of type t is the s-th etype into t (ascending)
 *   e_src_gid int64 [n_edges], e_eid int64 [n_edges], e_src int32 [n_edges] (src row)   */
typedef struct {
    const int64_t* dst_gid;
    const int64_t* src_gid;
    const int64_t* seg_ptr;
    const int64_t* e_src_gid;
    const int64_t* e_eid;
    const int32_t* e_src;
    int32_t num_slots; /* S */
} gsb_block_view;
gsb_status gsb_block_view_get(gsb_blocks_t b, const void* arena, int32_t layer, gsb_block_view* out);

/* Etype of slot s for node type t (-1 if none); host query. */
gsb_status gsb_slot_etype(gsb_graph_t g, int32_t ntype, int32_t slot, int32_t* etype);

/* Latched device error of the last sample (syncs): 0 = none, 1 = frontier not grouped by
 * type, 2 = gid out of range, 3 = capacity overflow. */
gsb_status gsb_blocks_poll_error(gsb_blocks_t b, void* arena, int32_t* code, void* stream);

/* Gather the input features of the sampled mini-batch (layer 0 src rows):
 * out: device [n_src(layer 0)][dim] in the feature dtype (capacity from
 * gsb_blocks_input_rows). */
gsb_status gsb_gather_block_inputs(gsb_blocks_t b, const void* arena, void* out, void* stream);
gsb_status gsb_blocks_input_rows(gsb_blocks_t b, int64_t* max_rows);
/* Row capacity of the dst rows of `layer` (for h_dst buffers). */
gsb_status gsb_blocks_dst_rows(gsb_blocks_t b, int32_t layer, int64_t* max_rows);

/* ======================================================================================
 * RGCN layer (P:L96 RGCN, ref [18]; §8(a) a7, a11):
 *   A_r[v] = (1/c_r(v)) sum_{sampled e: u->v in r} h_src[u]      (0 if c_r(v) = 0)
 *   Z_v    = sum_r A_r[v] W_r + h_src[self(v)] W_self + b ;  h_dst = ReLU(Z) or Z
 * computed as a per-relation segment mean followed by one grouped GEMM per dst type over
 * the concatenation Acat_v = [A_{r_0}[v] | ... | A_{r_{S_t-1}}[v] | h_src[self(v)]].
 * d_in must be a multiple of 32 and d_out a multiple of 4.
 * h_src == NULL (layer 0 only): source rows are read straight from the registered feature
 * tables by global id (in their dtype) -- the feature gather (§8(a) a5) fused into the
 * aggregation.  acat: device fp32 cache [gsb_layer_acat_floats] (kept for the backward).
 * ==================================================================================== */
gsb_status gsb_layer_acat_floats(gsb_blocks_t b, int32_t layer, int32_t d_in, int64_t* n_floats);

gsb_status gsb_rgcn_layer_fwd(gsb_blocks_t b, const void* arena, int32_t layer, const float* h_src, int32_t d_in,
                              const float* W, const float* bias, int32_t d_out, int32_t relu, float* h_dst,
                              float* acat, void* stream);
/* Same, with h_src of element type h_dtype (GSB_F32, or GSB_BF16 for gathered bf16 input
 * rows) and, when rowmap != NULL, source row r read at h_src[rowmap[r]] (rows delivered in
 * exchange order by gsb_bucket_by_owner's perm: the unpack is folded into the aggregation). */
gsb_status gsb_rgcn_layer_fwd_ex(gsb_blocks_t b, const void* arena, int32_t layer, const void* h_src, int32_t h_dtype,
                                 const int32_t* rowmap, int32_t d_in, const float* W, const float* bias, int32_t d_out,
                                 int32_t relu, float* h_dst, float* acat, void* stream);
/* The two halves of gsb_rgcn_layer_fwd_ex, for callers that schedule them apart:
 * gsb_rgcn_layer_agg fills acat (per-relation means + self rows; reads no parameter, so a
 *   pipelined caller runs it with the sampling of the next batch), gsb_rgcn_layer_gemm
 *   computes h_dst from acat.  fwd_ex = agg then gemm on one stream. */
gsb_status gsb_rgcn_layer_agg(gsb_blocks_t b, const void* arena, int32_t layer, const void* h_src, int32_t h_dtype,
                              const int32_t* rowmap, int32_t d_in, float* acat, void* stream);
gsb_status gsb_rgcn_layer_gemm(gsb_blocks_t b, const void* arena, int32_t layer, const float* acat, int32_t d_in,
                               const float* W, const float* bias, int32_t d_out, int32_t relu, float* h_dst,
                               void* stream);

/* Backward (analytic):  dZ = dh_dst * 1[h_dst > 0] (relu) or dh_dst;
 *   dW_r = sum_v A_r[v]^T dZ_v ; dW_self = sum_v h_src[self(v)]^T dZ_v ; db = sum_v dZ_v
 *   dh_src[u] += (1/c_r(v)) dZ_v W_r^T per sampled edge ; dh_src[self(v)] += dZ_v W_self^T
 * dW [R+1][d_in][d_out] and db [d_out] are overwritten; dh_src [n_src][d_in] is
 * overwritten when non-NULL (then dacat_ws [acat floats] is scratch).  With relu, dh_dst
 * is overwritten in place by dZ. */
gsb_status gsb_rgcn_layer_bwd(gsb_blocks_t b, const void* arena, int32_t layer, const float* h_dst,
                              float* dh_dst, const float* W, const float* acat, int32_t d_in, int32_t d_out,
                              int32_t relu, float* dW, float* db, float* dh_src, float* dacat_ws, void* stream);

/* ======================================================================================
 * Input encoder (§8(a) a6; "node input encoders handle node features"
 * featureless nodes) over the input rows of the sampled mini-batch (layer-0 src rows i,
 * type-grouped, count on the device):
 *   H0[i, :] = F_t[local(i), :] W_t     ntype t with W_in[t] != NULL: W_t device fp32
 *                                       [dim_t][d_out], features bf16, dim_t % 128 == 0
 *   H0[i, :] = F_t[local(i), :]         W_in[t] == NULL: frozen table, dim_t == d_out
 * W_in: host array [num_ntypes] of device pointers.  d_out % 128 == 0.  H0: device fp32
 * [gsb_blocks_input_rows][d_out] (the layer-0 h_src, GSB_F32).  The products run on tcgen05
 * bf16 MMAs with W (forward) / dH0 (backward) split into bf16 hi + lo (fp32-class accuracy).
 * ws: device scratch of gsb_encoder_ws_bytes (same W_in non-NULL pattern in every call).
 * Backward: dW_in[t] (device fp32 [dim_t][d_out], overwritten) = sum over input rows i of
 * type t of F_t[local(i)]^T dH0[i], for every t with W_in[t] != NULL; dH0 is layer 0's
 * dh_src (gsb_rgcn_layer_bwd).
 * ==================================================================================== */
gsb_status gsb_encoder_ws_bytes(gsb_blocks_t b, const float* const* W_in, int32_t d_out, size_t* bytes);
gsb_status gsb_encoder_fwd(gsb_blocks_t b, const void* arena, const float* const* W_in, int32_t d_out, float* H0,
                           void* ws, size_t ws_bytes, void* stream);
gsb_status gsb_encoder_bwd(gsb_blocks_t b, const void* arena, const float* const* W_in, const float* dH0,
                           int32_t d_out, float* const* dW_in, void* ws, size_t ws_bytes, void* stream);

/* Plain GEMM on the same tcgen05 3xTF32 path as the layers (single group), fp32 row-major:
 *   mode 0 (NN): C[M][N]  = A[M][K] B[K][N]        (K multiple of 32)
 *   mode 1 (NT): C[M][K]  = A[M][N] B[K][N]^T
 *   mode 2 (TN): C[K][N] += A[M][K]^T B[M][N]      (C accumulated; zero it first) */
gsb_status gsb_gemm(int32_t mode, const float* A, int64_t lda, const float* B, int64_t ldb, int64_t M, int32_t N,
                    int32_t K, float* C, int64_t ldc, void* stream);
/* Weight images (3xTF32 operand splits of weights, weights.cu): register W [slots][K][N]
 * (device fp32) with a caller-owned buffer of gsb_weight_images_bytes() bytes; refresh
 * recomputes the images of the given registered weights (call it after every update of W,
 * before the GEMMs that read it, in stream order -- inside a captured step is fine).  While a
 * weight is registered, the layer / decoder GEMMs whose B operand is that W read its images
 * through TMA instead of splitting W in every CTA.  Unregister before freeing W or the buffer. */
gsb_status gsb_weight_images_bytes(int32_t slots, int32_t K, int32_t N, size_t* bytes);
gsb_status gsb_weight_images_register(const float* W, int32_t slots, int32_t K, int32_t N, void* img,
                                      size_t img_bytes, void* stream);
gsb_status gsb_weight_images_unregister(const float* W);
gsb_status gsb_weight_images_refresh(const float* const* Ws, int32_t n, void* stream);
/* Same, with caller-provided images in W's own layout (hi, lo: device fp32 [slots][K][N],
 * N % 4 == 0, 16-B aligned) that the caller keeps current -- e.g. with gsb_adam_step_split
 * over a flat parameter buffer whose hi / lo twins hold the images.  No memset, no copy. */
gsb_status gsb_weight_images_register_split(const float* W, int32_t slots, int32_t K, int32_t N, float* hi,
                                            float* lo);

/* Tools: copies n (<= 256) globaltimer stamps recorded by CTA 0 of the last GEMM launched with
 * GSB_GEMM_DBG & 1024 ([role][64]: producer, MMA, splitters, epilogue; slot 63 = start). */
gsb_status gsb_gemm_trace(uint64_t* out, int32_t n);

/* ======================================================================================
 * Node-classification decoder + softmax cross-entropy (P:L477 ClassifyLossFunc, P:L489;
 * S:L405-408; §8(a) a8):  logits = h Wc + bc ; loss = mean_i(lse_i - logit_{i,y_i})
 *   y_i = labels[seed_gid[i] - label_gid_base].
 * Writes: logits_ws [n][ceil4(C)] (scratch, rows padded to a multiple of 4), loss (device fp32 scalar), dh [n][d], dWc [d][C],
 * dbc [C] (overwritten).  row_loss_ws: device fp32 [n + 640] scratch (row losses, then the
 * fused mean's block partials and ticket word); zero-fill it once before the first call.
 * dh may be NULL (no input gradient); dWc and dbc are both NULL (then logits_ws holds dlogits
 * for gsb_nc_loss_dw) or both set (computed on the library's side stream and joined into
 * `stream` before the call returns).  EINVAL on null inputs / bad dims.
 * ==================================================================================== */
gsb_status gsb_nc_loss(const float* h, int64_t n, int32_t d, const float* Wc, const float* bc, int32_t C,
                       const int32_t* labels, const int64_t* seed_gid, int64_t label_gid_base, float* logits_ws,
                       float* row_loss_ws, float* loss, float* dh, float* dWc, float* dbc, void* stream);
/* The decoder weight gradient on its own: dWc [d][C] = h^T dlogits, dbc [C] = column sums of
 * dlogits, where dlogits is what gsb_nc_loss left in logits_ws (same h, n, d, C; call it after
 * gsb_nc_loss in stream order -- e.g. on a second stream that waits for it -- when gsb_nc_loss
 * was given dWc = dbc = NULL).  Lets the caller overlap dWc with the layers' backward instead of
 * gsb_nc_loss joining it before returning.  pad_ws: optional device fp32 scratch of
 * d * ceil4(C) floats, 16-B aligned (NULL allowed): with C % 4 != 0 the GEMM's partials are
 * reduce-added into it by TMA and copied to dWc (else per-thread atomics into dWc).  dWc, dbc
 * overwritten; EINVAL on null / bad dims. */
gsb_status gsb_nc_loss_dw(const float* h, int64_t n, int32_t d, const float* logits_ws, int32_t C, float* dWc,
                          float* dbc, float* pad_ws, void* stream);

/* ======================================================================================
 * Full-graph inference (P:L393 layer-wise inference, P:L403 embedding
 * export).  Layer l of every node = the RGCN layer over its whole in-neighbourhood: sample a
 * chunk of consecutive gids with fanout ALL (gsb_sample, one layer), run gsb_rgcn_layer_fwd_ex
 * with h_src = the all-node table of layer l-1 and rowmap from gsb_blocks_input_rowmap (layer
 * 0: h_src NULL, the features are read by gid), writing the chunk's rows of layer l.
 * gsb_blocks_input_rowmap: rowmap[i] = src_gid[i] - gid_base for the first layer's input rows
 *   (device count); rowmap: device int32 [gsb_blocks_input_rows]; ids must fit int32.
 * gsb_nc_predict: logits = h Wc + bc (tcgen05 GEMM into logits_ws, device fp32 [n][C rounded up
 *   to 4]), pred[i] = argmax (lowest class on ties; pred nullable), and, when correct != NULL,
 *   *correct += #{i : pred[i] == labels[seed_gid[i] - label_gid_base]} (device uint64).
 *   d % 32 == 0.
 * ==================================================================================== */
gsb_status gsb_blocks_input_rowmap(gsb_blocks_t b, const void* arena, int64_t gid_base, int32_t* rowmap,
                                   void* stream);
gsb_status gsb_nc_predict(const float* h, int64_t n, int32_t d, const float* Wc, const float* bc, int32_t C,
                          const int32_t* labels, const int64_t* seed_gid, int64_t label_gid_base, float* logits_ws,
                          int32_t* pred, unsigned long long* correct, void* stream);

/* ======================================================================================
 * Learnable sparse embeddings for featureless ntypes ("GraphStorm
 * by default adds learnable embeddings on author nodes").  E: device fp32 [N_t][d] table of
 * ntype t (this GPU holds all of it), 16-byte aligned; d % 4 == 0.
 * gsb_sparse_emb_fwd: H0[i] = E[local(i)] for every layer-0 input row i of type t (run after
 *   gsb_encoder_fwd, which leaves those rows to the table).  H0 as in gsb_encoder_fwd.
 * gsb_sparse_adagrad: the gradient of E is dH0 on the touched rows only (a row copy; the
 *   input rows of one ntype are distinct); for each: state[r] += g^2,
 *   E[r] -= lr g / (sqrt(state[r]) + eps) (R-sparseopt: Adagrad, paper silent).  state:
 *   device fp32 [N_t][d], zero-initialised by the caller.  Untouched rows do not move.
 * ==================================================================================== */
gsb_status gsb_sparse_emb_fwd(gsb_blocks_t b, const void* arena, int32_t ntype, const float* E, int32_t d, float* H0,
                              void* stream);
gsb_status gsb_sparse_adagrad(gsb_blocks_t b, const void* arena, int32_t ntype, float* E, float* state,
                              const float* dH0, int32_t d, float lr, float eps, void* stream);

/* Tables partitioned over the N GPUs of one box (§8(e) with §8(f) f1; reading R-sparsedist:
 * the gradient of a row is the mean over ranks of the ranks' dEmb rows, and the owner takes
 * one Adagrad step with it).  bounds: host int64 [world+1], rank w owns local rows
 * [bounds[w], bounds[w+1]) of ntype t (bounds[0] = 0, bounds[world] = count of t), world <= 8.
 * Pointer arrays are host arrays of world device pointers: this rank's own buffers and the
 * peers' (IPC-mapped, gsb_ipc_open), each shard row-major [bounds[w+1]-bounds[w]][d] fp32.
 * gsb_sparse_emb_fwd_peers: H0[i] = E_w[x - bounds[w]] for every layer-0 input row i of type t
 *   (x its local id, w its owner): loads over NVLink.
 * gsb_sparse_emb_push: G_w[x - bounds[w]] += scale * dH0[i] (fp32 atomics, over NVLink for
 *   peers) and bit (x - bounds[w]) set in touched_w (uint32 words, bit k of word j = row
 *   32 j + k).  scale = 1 / world for the mean.  G and touched are zero between steps.
 * gsb_sparse_adagrad_apply (owner, on its own shard of n_rows rows): for every set bit,
 *   state += g^2, E -= lr g / (sqrt(state) + eps) with g the G row; then the G row and the bit
 *   are zeroed.  Untouched rows do not move.
 * Ordering: every rank's push must complete before any owner's apply, and every apply before
 * the next fwd reads the shards: the caller puts a cross-rank barrier (NCCL) between them. */
gsb_status gsb_sparse_emb_fwd_peers(gsb_blocks_t b, const void* arena, int32_t ntype, int32_t world,
                                    const int64_t* bounds, void* const* E, int32_t d, float* H0, void* stream);
gsb_status gsb_sparse_emb_push(gsb_blocks_t b, const void* arena, int32_t ntype, int32_t world, const int64_t* bounds,
                               void* const* G, void* const* touched, const float* dH0, int32_t d, float scale,
                               void* stream);
gsb_status gsb_sparse_adagrad_apply(float* E, float* state, float* G, uint32_t* touched, int64_t n_rows, int32_t d,
                                    float lr, float eps, void* stream);

/* ======================================================================================
 * Feature construction for featureless nodes (Eq. 1).
 *   F'_v = f(F_u, u in N(v)) with f = average (R-eq1): every in-edge u -> v of every stored
 *   etype whose dst type is `ntype` and whose src type is set in featured_mask (bit t = ntype
 *   t) counts once; F'_v = 0 when v has no such edge.  Local ids [first, first + count) of
 *   ntype; out: device fp32 [count][dim] (row-major), dim = the featured types' common width.
 *   A full sweep over the CSC (no sampling); features may be local or NVLink peer shards.
 * ==================================================================================== */
gsb_status gsb_construct_features(gsb_graph_t g, int32_t ntype, uint32_t featured_mask, int64_t first,
                                  int64_t count, float* out, int32_t dim, void* stream);

/* ======================================================================================
 * Link prediction (App. A; §8(a) a9, a10).
 * ==================================================================================== */
/* Joint negative sampling: positives in groups of K; group g draws K iid uniform
 * nodes of the dst type: neg[g*K + j] = gid_base + unif(Philox(g + group_base, j, step),
 * n_dst_nodes) (R-joint, R-rng).  neg: device int64 [ceil(n_pos/K)*K]. */
gsb_status gsb_joint_negatives(int64_t n_pos, int32_t K, int64_t n_dst_nodes, int64_t gid_base, uint64_t rng_seed,
                               uint32_t step, const uint32_t* step_dev, int64_t group_base, int64_t* neg,
                               void* stream);

/* Uniform negative sampling (App. A.2.1): every positive draws K
 * iid uniform nodes of the dst type: neg[i*K + j] = gid_base + unif(Philox(pos_base + i,
 * 0xFFE00000 | j, step), n_dst_nodes) (R-rng).  neg: device int64 [n_pos*K].
 * Local joint negative sampling is gsb_joint_negatives over the local partition's
 * range of the dst type (gid_base = first local gid, n_dst_nodes = local count).
 * In-batch negative sampling draws nothing: gsb_lp_score_ex neg_mode 1. */
gsb_status gsb_uniform_negatives(int64_t n_pos, int32_t K, int64_t n_dst_nodes, int64_t gid_base, uint64_t rng_seed,
                                 uint32_t step, const uint32_t* step_dev, int64_t pos_base, int64_t* neg,
                                 void* stream);

/* LP seed set (§8(a) a9): seeds = ascending unique(u ∪ v ∪ neg); iu/iv/ineg = row of
 * each u / v / neg in seeds.  seeds capacity 2*B + n_neg; *n_seeds_dev (device int64)
 * receives the count.  ws: device scratch of gsb_lp_seeds_bytes. */
gsb_status gsb_lp_seeds_bytes(int64_t B, int64_t n_neg, size_t* bytes);
gsb_status gsb_lp_seeds(const int64_t* u, const int64_t* v, int64_t B, const int64_t* neg, int64_t n_neg,
                        int64_t* seeds, int64_t* n_seeds_dev, int32_t* iu, int32_t* iv, int32_t* ineg, void* ws,
                        size_t ws_bytes, void* stream);

/* DistMult score (Eq. 3) + loss and its gradients.
 *   pos_i = sum_k H[iu_i,k] rel[k] H[iv_i,k] ; neg_ij = sum_k H[iu_i,k] rel[k] H[ineg_{g(i)K+j},k]
 *   loss_kind 0: contrastive Eq. 7 (R-lpmean); 1: cross entropy Eq. 4 (R-ce); mean over B.
 * H: device fp32 [n_rows][d] (last RGCN layer output over the LP seeds); scores: device
 * fp32 [B][1+K]; loss: device fp32 scalar; dH: device fp32 [n_rows][d] (overwritten,
 * n_rows_cap rows zeroed); drel [d] (overwritten); row_loss_ws: device fp32 [B]. */
gsb_status gsb_lp_score(const float* H, int64_t n_rows_cap, int32_t d, const int32_t* iu, const int32_t* iv,
                        const int32_t* ineg, int64_t B, int32_t K, const float* rel, int32_t loss_kind, float* scores,
                        float* row_loss_ws, float* loss, float* dH, float* drel, void* stream);

/* LP evaluation metric MRR (Tables 2 and 6 report it), reading R-mrr.
 *   scores: device fp32 [B][ld], row i = [pos_i, neg_i1 .. neg_iK] (the layout gsb_lp_score /
 *   gsb_lp_score_ex write, ld = 1 + K); rank_i = 1 + #{j: neg_ij > pos_i} + #{j: neg_ij ==
 *   pos_i} / 2 (compared in fp32); rr: device fp32 [B] receives 1 / rank_i; mrr: device fp32
 *   scalar, the mean of rr.  B >= 1, K >= 1, ld >= K + 1 (else GSB_ERR_ARG).  Caller-owned
 *   memory, asynchronous on stream. */
gsb_status gsb_lp_mrr(const float* scores, int64_t ld, int64_t B, int32_t K, float* rr, float* mrr, void* stream);

/* General LP score + loss (App. A).  Negative j of positive i is
 *   neg_mode 0 (sampled): row ineg[(i / group) * K + j]   (joint / local joint: group = K;
 *                          uniform: group = 1)
 *   neg_mode 1 (in-batch): row iv[j < i ? j : j + 1], K = B - 1 (ineg unused).
 * rel: DistMult relation vector (Eq. 3) or NULL for the dot product (Eq. 2; drel unused).
 * loss_kind 0 contrastive (Eq. 7), 1 cross entropy (Eq. 4, R-ce), 2 weighted cross entropy
 * (Eq. 5, R-wce): positive i's term times w[i] (device fp32 [B]); negatives weigh 1.
 * Other arguments and outputs as gsb_lp_score; scores: [B][1+K].
 * In-batch with B a multiple of 32 runs as dense contractions on the tensor cores:
 * S = (H[iu] o rel) H[iv]^T (B x B), the loss row-wise on S, then dS H[iv] and
 * dS^T (H[iu] o rel) (gsb_gemm, 3xTF32); ws: device scratch of gsb_lp_score_ws_bytes
 * (0 bytes otherwise; then ws may be NULL). */
gsb_status gsb_lp_score_ws_bytes(int64_t B, int32_t d, int32_t neg_mode, size_t* bytes);
gsb_status gsb_lp_score_ex(const float* H, int64_t n_rows_cap, int32_t d, const int32_t* iu, const int32_t* iv,
                           const int32_t* ineg, int64_t B, int32_t K, int32_t group, int32_t neg_mode,
                           const float* rel, int32_t loss_kind, const float* w, float* scores, float* row_loss_ws,
                           float* loss, float* dH, float* drel, void* ws, size_t ws_bytes, void* stream);

/* ======================================================================================
 * Partitioned feature store across GPUs (§8(e); P:L86 distributed tensors, P:L90 random
 * partitioning, P:L172 remote data movement).  Rank r owns local ids
 * [bounds[t][r], bounds[t][r+1]) of every ntype t and holds only those feature rows.  A
 * gather of arbitrary gids = bucket by owner -> NCCL all-to-all of ids (caller) ->
 * gsb_shard_gather on the owner -> all-to-all of rows (caller) -> gsb_rows_permute.
 * ==================================================================================== */
typedef struct gsb_partition* gsb_partition_t;
/* bounds: host int64 [num_ntypes][world+1], bounds[t][0] = 0, bounds[t][world] = count[t].
 * world <= 8. */
gsb_status gsb_partition_create(int32_t num_ntypes, const int64_t* ntype_count, int32_t world, int32_t rank,
                                const int64_t* bounds, gsb_partition_t* out);
gsb_status gsb_partition_destroy(gsb_partition_t p);
/* Register this rank's shard of ntype t: device rows (dim elements of dtype, 16-byte
 * aligned, row bytes a multiple of 16) for its owned local ids. */
gsb_status gsb_partition_set_shard(gsb_partition_t p, int32_t ntype, const void* rows, int32_t dim, int32_t dtype);
/* Owner bucketing (K11): for i < n (n = *n_dev if non-NULL, else n_cap): send_gid[perm[i]] =
 * gid[i] grouped by owner rank in rank order; send_counts: device int64 [world] (overwritten);
 * ws: device scratch of 8*world bytes.  Order inside a bucket is unspecified; perm is exact. */
gsb_status gsb_bucket_by_owner(gsb_partition_t p, const int64_t* gid, const int64_t* n_dev, int64_t n_cap,
                               int64_t* send_gid, int32_t* perm, int64_t* send_counts, void* ws, void* stream);
/* out[i, :] = own shard row of gid[i] (every gid must be owned by this rank); exact copy. */
gsb_status gsb_shard_gather(gsb_partition_t p, const int64_t* gid, int64_t n, void* out, void* stream);
/* out[i, :] = rows[perm[i], :] for i < n (n = *n_dev if non-NULL, else n_cap); rows of
 * row_bytes bytes (a multiple of 16), copied exactly. */
gsb_status gsb_rows_permute(const void* rows, int32_t row_bytes, const int32_t* perm, const int64_t* n_dev,
                            int64_t n_cap, void* out, void* stream);

/* ======================================================================================
 * Peer feature access over NVLink (§8(e); P:L86 distributed tensors).  Each rank keeps only
 * its node-ID range of every ntype; the other ranks' shards are mapped with CUDA IPC and the
 * fused layer-0 gather+aggregation (gsb_rgcn_layer_fwd with h_src = NULL) and gsb_gather read
 * every row from its owner's HBM directly -- no all-to-all, no host-synced sizes.
 * ==================================================================================== */
/* handle_out: 64 bytes (cudaIpcMemHandle_t of the allocation containing dev_ptr);
 * offset_out: dev_ptr's byte offset inside that allocation. */
gsb_status gsb_ipc_handle(const void* dev_ptr, void* handle_out, int64_t* offset_out);
/* Map another process's allocation (peer access enabled lazily); *dev_ptr_out = base + offset. */
gsb_status gsb_ipc_open(const void* handle, int64_t offset, void** dev_ptr_out);
gsb_status gsb_ipc_close(void* base_ptr);
/* Register ntype t's partitioned table: bounds host int64 [world+1] (local-id ranges, bounds[0]
 * = 0, bounds[world] = count), ptrs host [world] device pointers (own shard + IPC-mapped peer
 * shards), row-major [bounds[w+1]-bounds[w]][dim] of dtype (GSB_F32 / GSB_BF16).  world <= 8. */
/* Partitioned topology read over NVLink (§8(e); P:L86 sampling "on a distributed graph"):
 * rank w of `world` holds the CSC of the dst nodes it owns -- local ids [bounds[t][w],
 * bounds[t][w+1]) of every ntype t (bounds: host int64 [T][world+1]) -- built with
 * gsb_csc_build_range; indptr_w[w] / indices_w[w] are rank w's arrays of `etype` (this
 * process's own, or IPC-mapped peers' from gsb_ipc_open) and eid_base_w[w] their n_before.
 * After registration the sampler reads each dst's segment from its owner's HBM (keyed draws:
 * blocks identical to a whole-graph sampler, bit-exact).  table_dev: caller-owned device
 * memory of gsb_csc_peers_bytes() bytes, the same for every etype of g.  n_edges_total: the
 * etype's edge count over all shards (sizes the sampler's capacities).  Syncs stream. */
gsb_status gsb_csc_peers_bytes(size_t* bytes);
gsb_status gsb_graph_set_csc_peers(gsb_graph_t g, void* table_dev, int32_t etype, int32_t world,
                                   const int64_t* bounds, const int64_t* const* indptr_w,
                                   const int32_t* const* indices_w, const int64_t* eid_base_w, int64_t n_edges_total,
                                   void* stream);

gsb_status gsb_graph_set_feature_peers(gsb_graph_t g, int32_t ntype, int32_t world, const int64_t* bounds,
                                       const void* const* ptrs, int32_t dim, int32_t dtype);

/* ======================================================================================
 * Optimizer (paper silent, R-adam): Adam with bias correction over a flat
 * fp32 buffer of n parameters; t is the 1-based step.  In place on p, m, v.
 * ==================================================================================== */
gsb_status gsb_adam_step(float* p, const float* g, float* m, float* v, int64_t n, float lr, float beta1,
                         float beta2, float eps, int32_t t, const int32_t* t_dev, void* stream);
/* t_dev: optional device int32 overriding t (CUDA-graph replay). */
/* Adam that also writes the 3xTF32 split of the updated parameters (hi = rna_tf32(p),
 * lo = rna_tf32(p - hi); device fp32 [n], 16-B aligned): the weight images of
 * gsb_weight_images_register_split stay current without a separate pass.  Optionally (pad_hi
 * non-null) the split of one segment [pad_off, pad_off + pad_rows*pad_cols) is also written
 * row by row with stride pad_ld into pad_hi / pad_lo (the padded image of a weight whose own
 * row stride is not 16-B aligned, e.g. a 349-class decoder). */
gsb_status gsb_adam_step_split(float* p, const float* g, float* m, float* v, int64_t n, float lr, float beta1,
                               float beta2, float eps, int32_t t, const int32_t* t_dev, float* hi, float* lo,
                               int64_t pad_off, int32_t pad_rows, int32_t pad_cols, int32_t pad_ld, float* pad_hi,
                               float* pad_lo, void* stream);

/* Add `delta` to a device int32/uint32 counter (graph-capturable step advance). */
gsb_status gsb_counter_add(int32_t* counter, int32_t delta, void* stream);

/* Busy-wait kernel (profiling aid: lets the host enqueue a whole step before it runs). */
gsb_status gsb_spin(int64_t nanoseconds, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GSB_H_ */
