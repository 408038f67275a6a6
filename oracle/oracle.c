/*
 * oracle.c -- plain, slow, obviously-correct CPU reference for the RGCN mini-batch
 * train step of GraphStorm (arXiv 2406.06022).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2406_06022_b200/) never links, imports or executes it, and this file shares
 * no code, header, table or constant generator with the CUDA path.
 *
 * Citations: "P:Lnnn" = /root/reference/PAPER.md line nnn (section / equation);
 * "S:Lnnn" = SPEC.md line nnn; "R-x" = a reading recorded in DESIGN.md §Readings
 * (where the paper is silent or garbled; SURVEY.md §8(c) gives the proposals).
 *
 * Floating point: every float computation is done in double (fp64) from the fp32
 * input values widened exactly.  Integer work (Philox, index mapping, CSC, sampling,
 * relabel) is exact.
 *
 * Parity pins: see tests/test_oracle_*.py.  Functions without a pin: none (the
 * end-to-end loss trajectory on large configs is "parity unpinned").
 *
 * Threads: single-threaded by default.  oracle_set_threads(n) runs the layer's per-dst-row
 * loops (segment means, forward rows) and the weight gradient's per-(relation, input column)
 * rows on n OpenMP threads; every output element is still summed by one thread in the same
 * order as the serial loops, so the results are bit-identical for any n (used to time the
 * oracle on all host cores, bench.py cpu_baseline).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_MAXT 16
#define OR_MAXR 64

static int g_threads = 1;
void oracle_set_threads(int32_t n) { g_threads = n < 1 ? 1 : n; }
int32_t oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_num_procs();
#else
    return 1;
#endif
}

/* ======================================================================================
 * 1. Philox4x32-10 (Salmon et al., SC'11).  The paper is silent on the RNG (R-rng);
 *    counter-based so that every draw is a pure function of its key and counter.
 *    Pinned by the Random123 known-answer vectors (tests/golden/philox_kat.txt).
 * ==================================================================================== */
static void philox_round(uint32_t c[4], const uint32_t k[2]) {
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c[0];
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c[1] ^ k[0];
    uint32_t n1 = lo1;
    uint32_t n2 = hi0 ^ c[3] ^ k[1];
    uint32_t n3 = lo0;
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
}

void oracle_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t c[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
    uint32_t k[2] = {key[0], key[1]};
    for (int r = 0; r < 10; ++r) {
        if (r > 0) { k[0] += 0x9E3779B9u; k[1] += 0xBB67AE85u; }
        philox_round(c, k);
    }
    out[0] = c[0]; out[1] = c[1]; out[2] = c[2]; out[3] = c[3];
}

/* Uniform index in [0, n) from a 64-bit word: floor(x * n / 2^64) (R-rng, Lemire
 * multiply-high without rejection; bias <= n / 2^64). */
uint64_t oracle_unif_index(uint64_t x, uint64_t n) {
    return (uint64_t)(((unsigned __int128)x * (unsigned __int128)n) >> 64);
}

/* Keyed 64-bit draw: key = (seed lo, seed hi); u64 = (out[1] << 32) | out[0] (R-rng). */
uint64_t oracle_keyed_u64(uint64_t seed, uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3) {
    uint32_t ctr[4] = {c0, c1, c2, c3};
    uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    uint32_t o[4];
    oracle_philox4x32_10(ctr, key, o);
    return ((uint64_t)o[1] << 32) | (uint64_t)o[0];
}

/* Sampling draw i for (dst gid v, etype r, hop h, step s) (R-rng counter layout). */
static uint64_t sample_draw(uint64_t seed, int64_t v, int32_t r, int32_t hop, uint32_t i, uint32_t step) {
    uint32_t c2 = ((uint32_t)(r & 0xFFF) << 20) | ((uint32_t)(hop & 0xF) << 16) | (i & 0xFFFFu);
    return oracle_keyed_u64(seed, (uint32_t)(uint64_t)v, (uint32_t)((uint64_t)v >> 32), c2, step);
}

/* ======================================================================================
 * 2. Graph store: per-etype CSC over destination nodes ("distributed graph
 *    engine"; S:L240 edges owned by destination).  In-edges of a destination are kept
 *    in ascending (src, original COO index) order (R-csc).  eid = position in the CSC.
 * ==================================================================================== */
typedef struct { int32_t src; int64_t coo; } or_pair;

static int cmp_pair(const void* a, const void* b) {
    const or_pair* x = (const or_pair*)a;
    const or_pair* y = (const or_pair*)b;
    if (x->src != y->src) return x->src < y->src ? -1 : 1;
    if (x->coo != y->coo) return x->coo < y->coo ? -1 : 1;
    return 0;
}

/* keep may be NULL (keep all).  Returns the number of kept edges. */
int64_t oracle_build_csc(int64_t n_dst, int64_t n_edges, const int32_t* src, const int32_t* dst,
                         const uint8_t* keep, int64_t* indptr, int32_t* indices) {
    memset(indptr, 0, sizeof(int64_t) * (size_t)(n_dst + 1));
    for (int64_t e = 0; e < n_edges; ++e)
        if (!keep || keep[e]) indptr[dst[e] + 1] += 1;
    for (int64_t v = 0; v < n_dst; ++v) indptr[v + 1] += indptr[v];
    int64_t E = indptr[n_dst];
    or_pair* tmp = (or_pair*)malloc(sizeof(or_pair) * (size_t)(E > 0 ? E : 1));
    int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_dst > 0 ? n_dst : 1));
    for (int64_t v = 0; v < n_dst; ++v) fill[v] = indptr[v];
    for (int64_t e = 0; e < n_edges; ++e) {
        if (keep && !keep[e]) continue;
        int64_t p = fill[dst[e]]++;
        tmp[p].src = src[e];
        tmp[p].coo = e;
    }
    for (int64_t v = 0; v < n_dst; ++v) {
        int64_t a = indptr[v], b = indptr[v + 1];
        if (b - a > 1) qsort(tmp + a, (size_t)(b - a), sizeof(or_pair), cmp_pair);
    }
    for (int64_t p = 0; p < E; ++p) indices[p] = tmp[p].src;
    free(tmp);
    free(fill);
    return E;
}

typedef struct {
    int32_t T, R;
    int64_t node_off[OR_MAXT + 1];  /* gid = node_off[t] + local id (R-gid, type-major) */
    int32_t src_t[OR_MAXR], dst_t[OR_MAXR];
    const int64_t* indptr[OR_MAXR];
    const int32_t* indices[OR_MAXR];
} or_graph;

void* oracle_graph_new(int32_t T, const int64_t* counts, int32_t R, const int32_t* src_t, const int32_t* dst_t) {
    if (T > OR_MAXT || R > OR_MAXR) return NULL;
    or_graph* g = (or_graph*)calloc(1, sizeof(or_graph));
    g->T = T; g->R = R;
    g->node_off[0] = 0;
    for (int t = 0; t < T; ++t) g->node_off[t + 1] = g->node_off[t] + counts[t];
    for (int r = 0; r < R; ++r) { g->src_t[r] = src_t[r]; g->dst_t[r] = dst_t[r]; }
    return g;
}

void oracle_graph_set_csc(void* gp, int32_t r, const int64_t* indptr, const int32_t* indices) {
    or_graph* g = (or_graph*)gp;
    g->indptr[r] = indptr;
    g->indices[r] = indices;
}

void oracle_graph_free(void* g) { free(g); }

static int32_t type_of(const or_graph* g, int64_t gid) {
    for (int t = 0; t < g->T; ++t)
        if (gid < g->node_off[t + 1]) return t;
    return -1;
}

/* ======================================================================================
 * 3. Per-etype uniform fanout sampling, one hop (P:L58, P:L86 on-the-fly sampling;
 *    Fig. 4 fanout).  For every dst v (frontier order) and every
 *    etype r into type(v) (ascending r): choose min(f, deg') of the non-excluded in-edges
 *    uniformly without replacement (R-wor) with Floyd's algorithm (R-floyd), positions
 *    emitted in ascending order.  f < 0 means ALL.  deg' excludes the batch's LP target
 *    edges and their reverse twins (R-excl).
 * ==================================================================================== */
static int cmp_i64(const void* a, const void* b) {
    int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
    return x < y ? -1 : (x > y ? 1 : 0);
}

/* Floyd's algorithm (Bentley & Floyd, CACM 1987; R-floyd) given its f draws:
 *   S = {} ; for i = 0..f-1: j = n - f + i ; t = draws[i] (uniform in [0, j]) ;
 *            S += (t in S) ? {j} : {t}
 * On return s[0..f) holds S in ascending order (s may alias draws).  Returns f. */
int64_t oracle_floyd(int64_t n, int64_t f, int64_t* s) {
    int64_t* S = (int64_t*)malloc(sizeof(int64_t) * (size_t)(f > 0 ? f : 1));
    int64_t ns = 0;
    for (int64_t i = 0; i < f; ++i) {
        int64_t j = n - f + i;
        int64_t t = s[i];
        int in = 0;
        for (int64_t q = 0; q < ns; ++q) if (S[q] == t) { in = 1; break; }
        S[ns++] = in ? j : t;
    }
    qsort(S, (size_t)ns, sizeof(int64_t), cmp_i64);
    memcpy(s, S, sizeof(int64_t) * (size_t)ns);
    free(S);
    return ns;
}

/* Source gids excluded from dst v's segment in etype r: u for every batch positive
 * (u, v) of the target etype r*, and v' for every positive (v, v') when r is the reverse
 * etype of r* (R-excl).  Returns how many were written into out (caller capacity n_ex). */
static int64_t excluded_srcs(int32_t r, int64_t v_gid, const int64_t* ex_u, const int64_t* ex_v, int64_t n_ex,
                             int32_t ex_r, int32_t ex_rev, int64_t* out) {
    int64_t n = 0;
    for (int64_t k = 0; k < n_ex; ++k) {
        if (r == ex_r && ex_v[k] == v_gid) out[n++] = ex_u[k];
        else if (r == ex_rev && ex_u[k] == v_gid) out[n++] = ex_v[k];
    }
    return n;
}

/* Outputs (capacity cap edges):  seg_cnt[j*R + r] = #edges for (dst j, etype r);
 * per edge (j-major, r ascending, position ascending): src gid, eid (CSC position),
 * etype, dst row j.  Returns E, or -1 if cap is exceeded. */
int64_t oracle_sample_hop(const void* gp, const int64_t* dst_gid, int64_t n_dst, int32_t fanout,
                          uint64_t seed, uint32_t step, int32_t hop,
                          const int64_t* ex_u, const int64_t* ex_v, int64_t n_ex, int32_t ex_r, int32_t ex_rev,
                          int64_t* seg_cnt, int64_t* e_src_gid, int64_t* e_eid, int32_t* e_etype,
                          int64_t* e_dst_row, int64_t cap) {
    const or_graph* g = (const or_graph*)gp;
    int64_t E = 0;
    int64_t* pos = NULL; int64_t pos_cap = 0;     /* non-excluded positions of a segment */
    int64_t* S = NULL;   int64_t S_cap = 0;
    int64_t* xs = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_ex > 0 ? n_ex : 1));
    for (int64_t j = 0; j < n_dst; ++j) {
        int64_t v = dst_gid[j];
        int32_t t = type_of(g, v);
        int64_t vl = v - g->node_off[t];
        for (int32_t r = 0; r < g->R; ++r) {
            seg_cnt[j * g->R + r] = 0;
            if (g->dst_t[r] != t) continue;
            int64_t a = g->indptr[r][vl], b = g->indptr[r][vl + 1];
            int64_t deg = b - a;
            if (deg > pos_cap) { pos_cap = deg; pos = (int64_t*)realloc(pos, sizeof(int64_t) * (size_t)pos_cap); }
            int64_t nx = excluded_srcs(r, v, ex_u, ex_v, n_ex, ex_r, ex_rev, xs);
            int64_t degp = 0;
            for (int64_t p = 0; p < deg; ++p) {
                int64_t u = g->node_off[g->src_t[r]] + g->indices[r][a + p];
                int hit = 0;
                for (int64_t q = 0; q < nx; ++q) if (xs[q] == u) { hit = 1; break; }
                if (!hit) pos[degp++] = p;
            }
            int64_t take = (fanout < 0 || degp <= fanout) ? degp : fanout;
            if (E + take > cap) { free(pos); free(S); free(xs); return -1; }
            if (take == degp) {
                /* every non-excluded in-edge, ascending */
                for (int64_t q = 0; q < degp; ++q) {
                    int64_t p = pos[q];
                    e_src_gid[E] = g->node_off[g->src_t[r]] + g->indices[r][a + p];
                    e_eid[E] = a + p;
                    e_etype[E] = r;
                    e_dst_row[E] = j;
                    ++E;
                }
            } else {
                /* Floyd: draw i is unif(j_i + 1) with j_i = deg' - f + i */
                if (take > S_cap) { S_cap = take; S = (int64_t*)realloc(S, sizeof(int64_t) * (size_t)S_cap); }
                for (int64_t i = 0; i < take; ++i) {
                    int64_t jj = degp - take + i;
                    uint64_t x = sample_draw(seed, v, r, hop, (uint32_t)i, step);
                    S[i] = (int64_t)oracle_unif_index(x, (uint64_t)(jj + 1));
                }
                int64_t ns = oracle_floyd(degp, take, S);
                for (int64_t q = 0; q < ns; ++q) {
                    int64_t p = pos[S[q]];
                    e_src_gid[E] = g->node_off[g->src_t[r]] + g->indices[r][a + p];
                    e_eid[E] = a + p;
                    e_etype[E] = r;
                    e_dst_row[E] = j;
                    ++E;
                }
            }
            seg_cnt[j * g->R + r] = take;
        }
    }
    free(pos);
    free(S);
    free(xs);
    return E;
}

/* ======================================================================================
 * 4. Block construction / relabel (P:L484 blocks[i]; R-relabel).
 *    Per ntype t: src_list_t = [dst nodes of type t in frontier order]
 *                              ++ ascending-unique(sampled srcs of type t not in that list).
 *    Next frontier = concatenation over ascending t.  Edge src -> row in that list.
 * ==================================================================================== */
static int64_t find_i64(const int64_t* a, int64_t n, int64_t x) { /* linear: plain */
    for (int64_t i = 0; i < n; ++i) if (a[i] == x) return i;
    return -1;
}

typedef struct { int64_t key; int64_t idx; } or_kv;
static int cmp_kv(const void* a, const void* b) {
    const or_kv* x = (const or_kv*)a; const or_kv* y = (const or_kv*)b;
    if (x->key != y->key) return x->key < y->key ? -1 : 1;
    return x->idx < y->idx ? -1 : (x->idx > y->idx ? 1 : 0);
}

static int64_t bsearch_kv(const or_kv* a, int64_t n, int64_t key) {
    int64_t lo = 0, hi = n;
    while (lo < hi) { int64_t m = (lo + hi) / 2; if (a[m].key < key) lo = m + 1; else hi = m; }
    return (lo < n && a[lo].key == key) ? a[lo].idx : -1;
}

/* Returns n_src (or -1 on capacity).  Outputs: src_gid[n_src], e_src_row[E],
 * self_row[n_dst] (row of dst j in the src list), src_type_cnt[T] (rows per type). */
int64_t oracle_relabel(const void* gp, const int64_t* dst_gid, int64_t n_dst, const int64_t* e_src_gid, int64_t E,
                       int64_t* src_gid, int32_t* e_src_row, int64_t* self_row, int64_t* src_type_cnt, int64_t cap) {
    const or_graph* g = (const or_graph*)gp;
    int64_t n_src = 0;
    /* lookup table of (gid -> row) built as we go, searched by binary search over a sorted copy */
    or_kv* rows = (or_kv*)malloc(sizeof(or_kv) * (size_t)(n_dst + E + 1));
    int64_t nrows = 0;
    int64_t* cand = (int64_t*)malloc(sizeof(int64_t) * (size_t)(E + 1));
    or_kv* dsts = (or_kv*)malloc(sizeof(or_kv) * (size_t)(n_dst + 1));
    for (int64_t j = 0; j < n_dst; ++j) { dsts[j].key = dst_gid[j]; dsts[j].idx = j; }
    qsort(dsts, (size_t)n_dst, sizeof(or_kv), cmp_kv);
    for (int32_t t = 0; t < g->T; ++t) {
        int64_t start = n_src;
        for (int64_t j = 0; j < n_dst; ++j) {
            if (type_of(g, dst_gid[j]) != t) continue;
            if (n_src >= cap) goto fail;
            self_row[j] = n_src;
            src_gid[n_src] = dst_gid[j];
            rows[nrows].key = dst_gid[j]; rows[nrows].idx = n_src; ++nrows;
            ++n_src;
        }
        int64_t nc = 0;
        for (int64_t e = 0; e < E; ++e) {
            int64_t u = e_src_gid[e];
            if (type_of(g, u) != t) continue;
            if (bsearch_kv(dsts, n_dst, u) >= 0) continue;  /* already a dst node */
            cand[nc++] = u;
        }
        qsort(cand, (size_t)nc, sizeof(int64_t), cmp_i64);
        for (int64_t i = 0; i < nc; ++i) {
            if (i > 0 && cand[i] == cand[i - 1]) continue;
            if (n_src >= cap) goto fail;
            src_gid[n_src] = cand[i];
            rows[nrows].key = cand[i]; rows[nrows].idx = n_src; ++nrows;
            ++n_src;
        }
        src_type_cnt[t] = n_src - start;
    }
    qsort(rows, (size_t)nrows, sizeof(or_kv), cmp_kv);
    for (int64_t e = 0; e < E; ++e) e_src_row[e] = (int32_t)bsearch_kv(rows, nrows, e_src_gid[e]);
    free(rows); free(cand); free(dsts);
    (void)find_i64;
    return n_src;
fail:
    free(rows); free(cand); free(dsts);
    return -1;
}

/* ======================================================================================
 * 5. Feature gather by global id (P:L86 distributed tensors):
 *    out[i, :] = F_{t(i)}[gid_i - node_off[t(i)], :]  -- an exact copy.
 * ==================================================================================== */
void oracle_gather(const void* gp, const float* const* feat, int32_t dim, const int64_t* gid, int64_t n, float* out) {
    const or_graph* g = (const or_graph*)gp;
    for (int64_t i = 0; i < n; ++i) {
        int32_t t = type_of(g, gid[i]);
        const float* row = feat[t] + (size_t)(gid[i] - g->node_off[t]) * (size_t)dim;
        for (int32_t k = 0; k < dim; ++k) out[(size_t)i * dim + k] = row[k];
    }
}

/* ======================================================================================
 * 6. RGCN layer (P:L96 model zoo "RGCN", ref [18]; R-rgcn):
 *    Z_v = sum_r [c_r(v) > 0] (1/c_r(v)) sum_{e: u->v in r} h_u W_r + h_v W_self + b
 *    h'_v = ReLU(Z_v) on hidden layers, identity on the last.  c_r(v) = sampled count.
 *    W is (R+1, d_in, d_out) row-major, slot R = W_self.
 *    Edges are given as (dst row, etype, src row); self_row[v] = row of v among the srcs.
 * ==================================================================================== */
static void rel_counts(int64_t n_dst, int32_t R, const int64_t* e_dst, const int32_t* e_et, int64_t E, int64_t* c) {
    memset(c, 0, sizeof(int64_t) * (size_t)(n_dst * R));
    for (int64_t e = 0; e < E; ++e) c[e_dst[e] * R + e_et[e]] += 1;
}

/* A[v][r][:] = (1/c_r(v)) sum_{e into v in r} h_src[src(e)] ; zero when c_r(v) = 0 */
static void rel_means(int64_t n_dst, int32_t R, int32_t d_in, const int64_t* e_dst, const int32_t* e_et,
                      const int32_t* e_src, int64_t E, const int64_t* c, const double* h_src, double* A) {
    memset(A, 0, sizeof(double) * (size_t)(n_dst * R * d_in));
    /* edges come dst-row-major (j-major sampler order): the edges of row v are [off[v],
     * off[v+1]); each row's sums run in edge order whether the rows run serially or not */
    int64_t* off = (int64_t*)calloc((size_t)n_dst + 1, sizeof(int64_t));
    for (int64_t e = 0; e < E; ++e) off[e_dst[e] + 1] += 1;
    for (int64_t v = 0; v < n_dst; ++v) off[v + 1] += off[v];
    #pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int64_t v = 0; v < n_dst; ++v) {
        for (int64_t e = off[v]; e < off[v + 1]; ++e) {
            double* a = A + ((size_t)v * R + e_et[e]) * d_in;
            const double* h = h_src + (size_t)e_src[e] * d_in;
            for (int32_t k = 0; k < d_in; ++k) a[k] += h[k];
        }
        for (int32_t r = 0; r < R; ++r) {
            int64_t cc = c[v * R + r];
            if (cc == 0) continue;
            double* a = A + ((size_t)v * R + r) * d_in;
            for (int32_t k = 0; k < d_in; ++k) a[k] = a[k] / (double)cc;
        }
    }
    free(off);
}

/* Exposed for tests: the per-relation means A[v][r][:] and counts c[v][r] (section 6). */
void oracle_rgcn_means(int64_t n_dst, int32_t R, int32_t d_in, const int64_t* e_dst, const int32_t* e_et,
                       const int32_t* e_src, int64_t E, const double* h_src, int64_t* c, double* A) {
    rel_counts(n_dst, R, e_dst, e_et, E, c);
    rel_means(n_dst, R, d_in, e_dst, e_et, e_src, E, c, h_src, A);
}

void oracle_rgcn_fwd(int64_t n_dst, int32_t R, int32_t d_in, int32_t d_out,
                     const int64_t* e_dst, const int32_t* e_et, const int32_t* e_src, int64_t E,
                     const int64_t* self_row, const double* h_src, const double* W, const double* b,
                     int32_t relu, double* z, double* h_dst) {
    int64_t* c = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_dst * R + 1));
    double* A = (double*)malloc(sizeof(double) * (size_t)(n_dst * R * d_in + 1));
    rel_counts(n_dst, R, e_dst, e_et, E, c);
    rel_means(n_dst, R, d_in, e_dst, e_et, e_src, E, c, h_src, A);
    #pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int64_t v = 0; v < n_dst; ++v) {
        double* zv = z + (size_t)v * d_out;
        for (int32_t n = 0; n < d_out; ++n) zv[n] = b[n];
        for (int32_t r = 0; r <= R; ++r) {
            const double* a = (r < R) ? A + ((size_t)v * R + r) * d_in : h_src + (size_t)self_row[v] * d_in;
            if (r < R && c[v * R + r] == 0) continue;
            const double* Wr = W + (size_t)r * d_in * d_out;
            for (int32_t k = 0; k < d_in; ++k) {
                double ak = a[k];
                for (int32_t n = 0; n < d_out; ++n) zv[n] += ak * Wr[(size_t)k * d_out + n];
            }
        }
        for (int32_t n = 0; n < d_out; ++n)
            h_dst[(size_t)v * d_out + n] = (relu && zv[n] <= 0.0) ? 0.0 : zv[n];
    }
    free(c); free(A);
}

/* Backward of the layer above (S:L378-386 analytic grads):
 *   dZ = dh' * 1[Z > 0] (ReLU'(0) = 0) or dh' (identity);
 *   dW_r = sum_v A_r[v]^T dZ_v ; dW_self = sum_v h_{self(v)}^T dZ_v ; db = sum_v dZ_v ;
 *   dh_src[u] += (1/c_r(v)) dZ_v W_r^T per sampled edge u->v in r ;
 *   dh_src[self(v)] += dZ_v W_self^T.   dh_src may be NULL (frozen inputs). */
void oracle_rgcn_bwd(int64_t n_dst, int64_t n_src, int32_t R, int32_t d_in, int32_t d_out,
                     const int64_t* e_dst, const int32_t* e_et, const int32_t* e_src, int64_t E,
                     const int64_t* self_row, const double* h_src, const double* W, const double* z,
                     int32_t relu, const double* dh_dst, double* dW, double* db, double* dh_src) {
    int64_t* c = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n_dst * R + 1));
    double* A = (double*)malloc(sizeof(double) * (size_t)(n_dst * R * d_in + 1));
    double* dZ = (double*)malloc(sizeof(double) * (size_t)(n_dst * d_out + 1));
    double* tmp = (double*)malloc(sizeof(double) * (size_t)(d_in + 1));
    rel_counts(n_dst, R, e_dst, e_et, E, c);
    rel_means(n_dst, R, d_in, e_dst, e_et, e_src, E, c, h_src, A);
    for (int64_t i = 0; i < n_dst * d_out; ++i) dZ[i] = (relu && z[i] <= 0.0) ? 0.0 : dh_dst[i];
    memset(dW, 0, sizeof(double) * (size_t)(R + 1) * d_in * d_out);
    memset(db, 0, sizeof(double) * (size_t)d_out);
    if (dh_src) memset(dh_src, 0, sizeof(double) * (size_t)(n_src * d_in));
    /* dW_r[k][:] = sum over v (in row order) of a_v[k] * dZ_v: rows k of one relation in
     * blocks of 16 per thread, every element summed over v in ascending order */
    const int32_t nkb = (d_in + 15) / 16;
    #pragma omp parallel for schedule(static) num_threads(g_threads)
    for (int64_t rb = 0; rb < (int64_t)(R + 1) * nkb; ++rb) {
        const int32_t r = (int32_t)(rb / nkb), k0 = (int32_t)(rb % nkb) * 16;
        const int32_t k1 = k0 + 16 < d_in ? k0 + 16 : d_in;
        double* dWr = dW + (size_t)r * d_in * d_out;
        for (int64_t v = 0; v < n_dst; ++v) {
            if (r < R && c[v * R + r] == 0) continue;
            const double* a = (r < R) ? A + ((size_t)v * R + r) * d_in : h_src + (size_t)self_row[v] * d_in;
            const double* g = dZ + (size_t)v * d_out;
            for (int32_t k = k0; k < k1; ++k) {
                const double ak = a[k];
                for (int32_t n = 0; n < d_out; ++n) dWr[(size_t)k * d_out + n] += ak * g[n];
            }
        }
    }
    for (int64_t v = 0; v < n_dst; ++v) {
        const double* g = dZ + (size_t)v * d_out;
        for (int32_t n = 0; n < d_out; ++n) db[n] += g[n];
        if (dh_src) {
            /* self term */
            const double* Ws = W + (size_t)R * d_in * d_out;
            double* ds = dh_src + (size_t)self_row[v] * d_in;
            for (int32_t k = 0; k < d_in; ++k) {
                double s = 0.0;
                for (int32_t n = 0; n < d_out; ++n) s += g[n] * Ws[(size_t)k * d_out + n];
                ds[k] += s;
            }
        }
    }
    if (dh_src) {
        for (int64_t e = 0; e < E; ++e) {
            int64_t v = e_dst[e];
            int32_t r = e_et[e];
            const double* g = dZ + (size_t)v * d_out;
            const double* Wr = W + (size_t)r * d_in * d_out;
            double inv = 1.0 / (double)c[v * R + r];
            for (int32_t k = 0; k < d_in; ++k) {
                double s = 0.0;
                for (int32_t n = 0; n < d_out; ++n) s += g[n] * Wr[(size_t)k * d_out + n];
                tmp[k] = s * inv;
            }
            double* du = dh_src + (size_t)e_src[e] * d_in;
            for (int32_t k = 0; k < d_in; ++k) du[k] += tmp[k];
        }
    }
    free(c); free(A); free(dZ); free(tmp);
}

/* ======================================================================================
 * 7. Node-classification decoder + softmax cross-entropy (P:L477 ClassifyLossFunc,
 *    P:L489; R-ncloss batch mean):
 *    logits = h Wc + bc ; loss = mean_i (logsumexp(logits_i) - logits_i[y_i]) ;
 *    dlogits = (softmax - onehot) / n ; dh = dlogits Wc^T ; dWc = h^T dlogits ; dbc = sum.
 * ==================================================================================== */
double oracle_nc_loss(int64_t n, int32_t d, int32_t C, const double* h, const double* Wc, const double* bc,
                      const int32_t* y, double* logits, double* dh, double* dWc, double* dbc) {
    double loss = 0.0;
    double* p = (double*)malloc(sizeof(double) * (size_t)C);
    if (dWc) memset(dWc, 0, sizeof(double) * (size_t)d * C);
    if (dbc) memset(dbc, 0, sizeof(double) * (size_t)C);
    for (int64_t i = 0; i < n; ++i) {
        double* lg = logits + (size_t)i * C;
        for (int32_t c = 0; c < C; ++c) {
            double s = bc[c];
            for (int32_t k = 0; k < d; ++k) s += h[(size_t)i * d + k] * Wc[(size_t)k * C + c];
            lg[c] = s;
        }
        double mx = lg[0];
        for (int32_t c = 1; c < C; ++c) if (lg[c] > mx) mx = lg[c];
        double se = 0.0;
        for (int32_t c = 0; c < C; ++c) se += exp(lg[c] - mx);
        double lse = mx + log(se);
        loss += lse - lg[y[i]];
        for (int32_t c = 0; c < C; ++c) p[c] = (exp(lg[c] - lse) - (c == y[i] ? 1.0 : 0.0)) / (double)n;
        if (dh)
            for (int32_t k = 0; k < d; ++k) {
                double s = 0.0;
                for (int32_t c = 0; c < C; ++c) s += p[c] * Wc[(size_t)k * C + c];
                dh[(size_t)i * d + k] = s;
            }
        if (dWc)
            for (int32_t k = 0; k < d; ++k)
                for (int32_t c = 0; c < C; ++c) dWc[(size_t)k * C + c] += h[(size_t)i * d + k] * p[c];
        if (dbc)
            for (int32_t c = 0; c < C; ++c) dbc[c] += p[c];
    }
    free(p);
    return loss / (double)n;
}

/* ======================================================================================
 * 8. Joint negative sampling (App. A.2.1): positives are taken in groups of K;
 *    each group g draws K nodes of dst_t uniformly (iid, with replacement, R-joint),
 *    shared by the group's positives.  ceil(n_pos/K)*K draws; the last partial
 *    group draws a fresh K-set.  Draw j of group g uses counter
 *    (g lo, g hi, 0xFFF00000 | j, step) (R-rng).  neg[g*K + j] = gid_base + index.
 * ==================================================================================== */
int64_t oracle_joint_negatives(int64_t n_pos, int32_t K, int64_t n_dst_nodes, int64_t gid_base,
                               uint64_t seed, uint32_t step, int64_t group_base, int64_t* neg) {
    int64_t G = (n_pos + K - 1) / K;
    for (int64_t g = 0; g < G; ++g) {
        int64_t gg = group_base + g;
        for (int32_t j = 0; j < K; ++j) {
            uint64_t x = oracle_keyed_u64(seed, (uint32_t)(uint64_t)gg, (uint32_t)((uint64_t)gg >> 32),
                                          0xFFF00000u | ((uint32_t)j & 0xFFFFu), step);
            neg[g * K + j] = gid_base + (int64_t)oracle_unif_index(x, (uint64_t)n_dst_nodes);
        }
    }
    return G * K;
}

/* ======================================================================================
 * 8b. Uniform negative sampling (App. A.2.1): every positive i draws K nodes of
 *     dst_t uniformly (iid, with replacement): N*K draws in total.  Draw j of positive p =
 *     pos_base + i uses counter (p lo, p hi, 0xFFE00000 | j, step) (R-rng; etype id 0xFFE
 *     is reserved for uniform negatives as 0xFFF is for joint ones).
 *     neg[i*K + j] = gid_base + index.
 *     Local joint negative sampling is joint sampling with gid_base / n_dst_nodes
 *     restricted to the local partition's range of dst_t: no separate routine.
 *     In-batch negative sampling draws nothing (see oracle_lp_loss_ex, mode 1).
 * ==================================================================================== */
int64_t oracle_uniform_negatives(int64_t n_pos, int32_t K, int64_t n_dst_nodes, int64_t gid_base,
                                 uint64_t seed, uint32_t step, int64_t pos_base, int64_t* neg) {
    for (int64_t i = 0; i < n_pos; ++i) {
        int64_t p = pos_base + i;
        for (int32_t j = 0; j < K; ++j) {
            uint64_t x = oracle_keyed_u64(seed, (uint32_t)(uint64_t)p, (uint32_t)((uint64_t)p >> 32),
                                          0xFFE00000u | ((uint32_t)j & 0xFFFFu), step);
            neg[i * K + j] = gid_base + (int64_t)oracle_unif_index(x, (uint64_t)n_dst_nodes);
        }
    }
    return n_pos * K;
}

/* ======================================================================================
 * 9. Link-prediction score (App. A.1) and losses (App. A.2):
 *    score(u, x) = sum_k u[k] rel[k] x[k]   DistMult, Eq. 3
 *                = sum_k u[k] x[k]          dot product, Eq. 2, rel == NULL
 *    Positive i scores (hu_i, hv_i); its K negatives replace the destination:
 *      mode 0 (sampled negatives, shared by groups of `group` positives): negative j of
 *             positive i is hn row (i / group) * K + j.  Joint / local joint: group = K
 *             (P:L356-357); uniform: group = 1.
 *      mode 1 (in-batch): the negatives of positive i are the destinations of the
 *             other positives, in batch order: j -> hv row (j < i ? j : j + 1); K = B - 1.
 *    loss_kind 0: contrastive Eq. 7: l_i = -log(exp(pos_i)/sum_{all 1+K} exp(s))
 *    loss_kind 1: cross entropy Eq. 4 (garbled; R-ce): per edge
 *       -[y ln sigma(s) + (1-y) ln(1 - sigma(s))], mean over the 1+K edges, then over i.
 *    loss_kind 2: weighted cross entropy Eq. 5 (R-wce): as 1 with the positive
 *       edge's term multiplied by its weight w[i]; negatives weigh 1.
 *    Batch mean over positives (R-lpmean).  scores[i*(1+K)+0] = pos, [1+j] = neg_ij.
 *    Gradients: dhu (B,d), dhv (B,d), dhn (rows of hn, d; mode 0 only; a row accumulates
 *    over the positives that share it), drel (d; DistMult only).
 * ==================================================================================== */
static double log_sigmoid(double s) { return s >= 0 ? -log1p(exp(-s)) : s - log1p(exp(s)); }
static double sigmoid(double s) { return s >= 0 ? 1.0 / (1.0 + exp(-s)) : exp(s) / (1.0 + exp(s)); }

double oracle_lp_loss_ex(int64_t B, int32_t K, int32_t group, int32_t mode, int32_t d, const double* hu,
                         const double* hv, const double* hn, int64_t n_hn, const double* rel, int32_t loss_kind,
                         const double* w, double* scores, double* dhu, double* dhv, double* dhn, double* drel) {
    double loss = 0.0;
    double* ds = (double*)malloc(sizeof(double) * (size_t)(K + 1));
    memset(dhu, 0, sizeof(double) * (size_t)(B * d));
    memset(dhv, 0, sizeof(double) * (size_t)(B * d));
    if (dhn) memset(dhn, 0, sizeof(double) * (size_t)(n_hn * d));
    if (drel) memset(drel, 0, sizeof(double) * (size_t)d);
    for (int64_t i = 0; i < B; ++i) {
        double* sc = scores + (size_t)i * (K + 1);
        const double* u = hu + (size_t)i * d;
        const double* v = hv + (size_t)i * d;
        double s = 0.0;
        for (int32_t k = 0; k < d; ++k) s += u[k] * (rel ? rel[k] : 1.0) * v[k];
        sc[0] = s;
        for (int32_t j = 0; j < K; ++j) {
            const double* nn = mode == 0 ? hn + ((size_t)(i / group) * K + j) * d
                                         : hv + (size_t)(j < i ? j : j + 1) * d;
            double t = 0.0;
            for (int32_t k = 0; k < d; ++k) t += u[k] * (rel ? rel[k] : 1.0) * nn[k];
            sc[1 + j] = t;
        }
        if (loss_kind == 0) {
            double mx = sc[0];
            for (int32_t j = 1; j <= K; ++j) if (sc[j] > mx) mx = sc[j];
            double se = 0.0;
            for (int32_t j = 0; j <= K; ++j) se += exp(sc[j] - mx);
            double lse = mx + log(se);
            loss += lse - sc[0];
            for (int32_t j = 0; j <= K; ++j) ds[j] = (exp(sc[j] - lse) - (j == 0 ? 1.0 : 0.0)) / (double)B;
        } else {
            double wi = (loss_kind == 2) ? w[i] : 1.0;
            double li = -wi * log_sigmoid(sc[0]);
            ds[0] = wi * (sigmoid(sc[0]) - 1.0) / (double)(K + 1) / (double)B;
            for (int32_t j = 1; j <= K; ++j) {
                li += -log_sigmoid(-sc[j]);
                ds[j] = sigmoid(sc[j]) / (double)(K + 1) / (double)B;
            }
            loss += li / (double)(K + 1);
        }
        /* chain rule through s = sum_k u r x */
        for (int32_t k = 0; k < d; ++k) {
            double r = rel ? rel[k] : 1.0;
            dhu[(size_t)i * d + k] += ds[0] * r * v[k];
            dhv[(size_t)i * d + k] += ds[0] * u[k] * r;
            if (drel) drel[k] += ds[0] * u[k] * v[k];
        }
        for (int32_t j = 0; j < K; ++j) {
            const double* nn;
            double* dn;
            if (mode == 0) {
                nn = hn + ((size_t)(i / group) * K + j) * d;
                dn = dhn + ((size_t)(i / group) * K + j) * d;
            } else {
                nn = hv + (size_t)(j < i ? j : j + 1) * d;
                dn = dhv + (size_t)(j < i ? j : j + 1) * d;
            }
            for (int32_t k = 0; k < d; ++k) {
                double r = rel ? rel[k] : 1.0;
                dhu[(size_t)i * d + k] += ds[1 + j] * r * nn[k];
                dn[k] += ds[1 + j] * u[k] * r;
                if (drel) drel[k] += ds[1 + j] * u[k] * nn[k];
            }
        }
    }
    free(ds);
    return loss / (double)B;
}

/* Joint negatives + DistMult (the §8(a) a10 default): oracle_lp_loss_ex with group = K. */
double oracle_lp_loss(int64_t B, int32_t K, int32_t d, const double* hu, const double* hv, const double* hn,
                      const double* rel, int32_t loss_kind, double* scores,
                      double* dhu, double* dhv, double* dhn, double* drel) {
    int64_t G = (B + K - 1) / K;
    return oracle_lp_loss_ex(B, K, K, 0, d, hu, hv, hn, G * K, rel, loss_kind, NULL, scores, dhu, dhv, dhn, drel);
}

/* ======================================================================================
 * 10. Optimizers (paper silent, R-adam): Adam beta1 0.9, beta2 0.999,
 *     eps 1e-8 with bias correction; SGD p -= lr g.
 * ==================================================================================== */
void oracle_adam(int64_t n, double* p, const double* g, double* m, double* v,
                 double lr, double b1, double b2, double eps, int32_t t) {
    double c1 = 1.0 - pow(b1, (double)t);
    double c2 = 1.0 - pow(b2, (double)t);
    for (int64_t i = 0; i < n; ++i) {
        m[i] = b1 * m[i] + (1.0 - b1) * g[i];
        v[i] = b2 * v[i] + (1.0 - b2) * g[i] * g[i];
        double mh = m[i] / c1;
        double vh = v[i] / c2;
        p[i] -= lr * mh / (sqrt(vh) + eps);
    }
}

/* Sparse Adagrad for learnable embedding tables (paper silent on the
 * optimizer, R-sparseopt): for each touched row r with gradient row g (rows distinct):
 *    state[r] += g*g ;  E[r] -= lr * g / (sqrt(state[r]) + eps)    (elementwise)
 * Untouched rows and their state are left as they are. */
void oracle_sparse_adagrad(int64_t n_rows, int32_t d, const int64_t* rows, const double* g, double* E,
                           double* state, double lr, double eps) {
    for (int64_t i = 0; i < n_rows; ++i) {
        double* e = E + (size_t)rows[i] * d;
        double* st = state + (size_t)rows[i] * d;
        const double* gi = g + (size_t)i * d;
        for (int32_t k = 0; k < d; ++k) {
            st[k] += gi[k] * gi[k];
            e[k] -= lr * gi[k] / (sqrt(st[k]) + eps);
        }
    }
}

void oracle_sgd(int64_t n, double* p, const double* g, double lr) {
    for (int64_t i = 0; i < n; ++i) p[i] -= lr * g[i];
}
