/* SPDX-License-Identifier: Apache-2.0
 *
 * TEST INFRASTRUCTURE ONLY — CPU restatement oracle of the reference dcpsim
 * decode path (see dcp_oracle.h).  Plain C11 + OpenMP.  Each function cites the
 * reference lines it restates (relative to /root/reference/proj).  The product
 * never links this file; tests compare the product against it and against the
 * reference itself (oracle/_ref).
 */
#include "dcp_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

/* error codes shared with include/dcp_capi.h */
enum { E_FRAMES = -1, E_UNKNOWN_REQ = -2, E_UNKNOWN_PAGE = -3, E_INCONS = -4, E_SHAPE = -5,
       E_EMPTY = -6, E_CONFIG = -7 };

static int64_t pages_for(int64_t tokens, int64_t page) { /* types.hpp:100-102 */
    return (tokens + page - 1) / page;
}

/* ======================================================================
 * Attention math — attn_merge.hpp:25-100, attn_merge.cpp:9-46
 * ====================================================================== */

/* shard_attention<double>: attn_merge.hpp:53-82.  Serial online softmax over
 * keys in order; the running max is raised (and acc/denom rescaled) only when
 * a strictly larger score appears (hpp:68-74); lse = max + log(denom) (hpp:80). */
int dcpora_shard_attention_f64(const double* q, const double* k, const double* v, int64_t len,
                               int d, double scale, double* out, double* lse) {
    if (len < 1) return E_EMPTY; /* hpp:57 */
    double mx = -INFINITY, den = 0.0;
    for (int i = 0; i < d; ++i) out[i] = 0.0;
    for (int64_t j = 0; j < len; ++j) {
        const double* kj = k + j * d;
        const double* vj = v + j * d;
        double s = 0.0;
        for (int i = 0; i < d; ++i) s += kj[i] * q[i];
        s *= scale;
        if (s > mx) {
            const double shrink = exp(mx - s);
            den *= shrink;
            for (int i = 0; i < d; ++i) out[i] *= shrink;
            mx = s;
        }
        const double w = exp(s - mx);
        den += w;
        for (int i = 0; i < d; ++i) out[i] += w * vj[i];
    }
    for (int i = 0; i < d; ++i) out[i] /= den;
    *lse = mx + log(den);
    return 0;
}

int dcpora_shard_attention_f32(const float* q, const float* k, const float* v, int64_t len, int d,
                               float scale, float* out, float* lse) {
    if (len < 1) return E_EMPTY;
    float mx = -INFINITY, den = 0.0f;
    for (int i = 0; i < d; ++i) out[i] = 0.0f;
    for (int64_t j = 0; j < len; ++j) {
        const float* kj = k + j * d;
        const float* vj = v + j * d;
        float s = 0.0f;
        for (int i = 0; i < d; ++i) s += kj[i] * q[i];
        s *= scale;
        if (s > mx) {
            const float shrink = expf(mx - s);
            den *= shrink;
            for (int i = 0; i < d; ++i) out[i] *= shrink;
            mx = s;
        }
        const float w = expf(s - mx);
        den += w;
        for (int i = 0; i < d; ++i) out[i] += w * vj[i];
    }
    for (int i = 0; i < d; ++i) out[i] /= den;
    *lse = mx + logf(den);
    return 0;
}

/* reference_attention<double>: attn_merge.hpp:25-50 (same recurrence, no LSE). */
int dcpora_reference_attention_f64(const double* q, const double* k, const double* v, int64_t len,
                                   int d, double scale, double* out) {
    double lse;
    if (len < 1) { /* the reference divides 0/0 here; mirror "no keys" as NaN */
        for (int i = 0; i < d; ++i) out[i] = NAN;
        return 0;
    }
    return dcpora_shard_attention_f64(q, k, v, len, d, scale, out, &lse);
}

/* lse_merge<double>: attn_merge.hpp:86-100.  m = max lse; w_k = exp(lse_k - m);
 * out = sum w_k o_k / sum w_k, folded in list order. */
int dcpora_lse_merge_f64(int n, const double* outs, const double* lses, int d, double* out) {
    if (n < 1) return E_EMPTY; /* hpp:88 */
    double m = -INFINITY, ws = 0.0;
    for (int k = 0; k < n; ++k) m = lses[k] > m ? lses[k] : m;
    for (int i = 0; i < d; ++i) out[i] = 0.0;
    for (int k = 0; k < n; ++k) {
        const double w = exp(lses[k] - m);
        ws += w;
        for (int i = 0; i < d; ++i) out[i] += w * outs[(size_t)k * d + i];
    }
    for (int i = 0; i < d; ++i) out[i] /= ws;
    return 0;
}

static int lse_merge_f32(int n, const float* outs, const float* lses, int d, float* out) {
    if (n < 1) return E_EMPTY;
    float m = -INFINITY, ws = 0.0f;
    for (int k = 0; k < n; ++k) m = lses[k] > m ? lses[k] : m;
    for (int i = 0; i < d; ++i) out[i] = 0.0f;
    for (int k = 0; k < n; ++k) {
        const float w = expf(lses[k] - m);
        ws += w;
        for (int i = 0; i < d; ++i) out[i] += w * outs[(size_t)k * d + i];
    }
    for (int i = 0; i < d; ++i) out[i] /= ws;
    return 0;
}

/* merge_impl / partition_impl: attn_merge.cpp:9-46.  bounds are exclusive
 * shard ends; zero-width shards are skipped (cpp:27) and dropped before the
 * merge (cpp:41-44); the merge runs in shard-index order. */
int dcpora_sharded_attention_merge_f64(const double* q, const double* k, const double* v,
                                       int64_t len, int d, double scale, const int64_t* bounds,
                                       int nb, double* out) {
    (void)len;
    double* outs = malloc(sizeof(double) * (size_t)nb * d);
    double* lses = malloc(sizeof(double) * (size_t)nb);
    int live = 0, rc = 0;
    int64_t start = 0;
    for (int i = 0; i < nb && !rc; ++i) {
        const int64_t lo = start, hi = bounds[i];
        start = bounds[i];
        if (hi <= lo) continue;
        rc = dcpora_shard_attention_f64(q, k + lo * d, v + lo * d, hi - lo, d, scale,
                                        outs + (size_t)live * d, lses + live);
        ++live;
    }
    if (!rc) rc = dcpora_lse_merge_f64(live, outs, lses, d, out);
    free(outs);
    free(lses);
    return rc;
}

int dcpora_sharded_attention_merge_f32(const float* q, const float* k, const float* v, int64_t len,
                                       int d, float scale, const int64_t* bounds, int nb,
                                       float* out) {
    (void)len;
    float* outs = malloc(sizeof(float) * (size_t)nb * d);
    float* lses = malloc(sizeof(float) * (size_t)nb);
    int live = 0, rc = 0;
    int64_t start = 0;
    for (int i = 0; i < nb && !rc; ++i) {
        const int64_t lo = start, hi = bounds[i];
        start = bounds[i];
        if (hi <= lo) continue;
        rc = dcpora_shard_attention_f32(q, k + lo * d, v + lo * d, hi - lo, d, scale,
                                        outs + (size_t)live * d, lses + live);
        ++live;
    }
    if (!rc) rc = lse_merge_f32(live, outs, lses, d, out);
    free(outs);
    free(lses);
    return rc;
}

static double bf16_to_f64(uint16_t x) {
    const uint32_t u = (uint32_t)x << 16;
    float f;
    memcpy(&f, &u, 4);
    return (double)f;
}

/* shard_attention<double> (hpp:53-82) applied per (shard, q-head) to the keys
 * of a paged KV layout: the shard's tokens are the valid slots of its pages in
 * logical page order (page_table.cpp:9-49 lays pages out in token order). */
/* Paged decode over a pool whose elements are bf16 (elem_bytes 2, widened exactly) or fp32
 * (elem_bytes 4, the reference's production precision, attn_merge.cpp:64-77): per (shard,
 * q-head) the reference's shard_attention<double> over the shard's tokens in page order. */
static double elem_f64(const void* base, size_t i, int elem_bytes) {
    if (elem_bytes == 4) return (double)((const float*)base)[i];
    return bf16_to_f64(((const uint16_t*)base)[i]);
}

int dcpora_paged_decode_attn_any_f64(int nshards, int hq, int hkv, int d, int page_size, int elem_bytes,
                                     const void* q_in, const void* pool_in, const int32_t* block_table,
                                     const int32_t* cu_pages, const int64_t* shard_len, const uint8_t* page_fill,
                                     double scale, double* out, double* lse, int threads) {
    /* Streams the shard's pages instead of gathering them: per (shard, kv-head) every token's
     * K and V rows are widened once and fed to the recurrence of each of the group's q-heads
     * in token order -- per q-head the exact arithmetic sequence of shard_attention<double>
     * (attn_merge.hpp:62-80, dcpora_shard_attention_f64), so results are bit-identical. */
    const int group = hq / hkv;
    const size_t head_elems = (size_t)page_size * d;
    const size_t frame_elems = 2 * (size_t)hkv * head_elems;
#pragma omp parallel for schedule(dynamic) num_threads(threads > 0 ? threads : 1)
    for (int64_t w = 0; w < (int64_t)nshards * hkv; ++w) {
        const int r = (int)(w / hkv), j = (int)(w % hkv);
        const int p0 = cu_pages[r], p1 = cu_pages[r + 1];
        double* qd = malloc(sizeof(double) * (size_t)group * d);
        double* kd = malloc(sizeof(double) * d);
        double* vd = malloc(sizeof(double) * d);
        double* mx = malloc(sizeof(double) * group);
        double* den = malloc(sizeof(double) * group);
        for (int g = 0; g < group; ++g) {
            const int h = j * group + g;
            for (int i = 0; i < d; ++i) qd[(size_t)g * d + i] = elem_f64(q_in, ((size_t)r * hq + h) * d + i, elem_bytes);
            double* o = out + ((size_t)r * hq + h) * d;
            for (int i = 0; i < d; ++i) o[i] = 0.0;
            mx[g] = -INFINITY;
            den[g] = 0.0;
        }
        int64_t ntok = 0;
        for (int p = p0; p < p1; ++p) {
            const int64_t rem = shard_len[r] - (int64_t)(p - p0) * page_size;
            const int fill = page_fill ? page_fill[p] : (int)(rem < page_size ? rem : page_size);
            const size_t kp = (size_t)block_table[p] * frame_elems + (size_t)j * head_elems;
            const size_t vp = kp + (size_t)hkv * head_elems;
            for (int t = 0; t < fill; ++t, ++ntok) {
                for (int i = 0; i < d; ++i) {
                    kd[i] = elem_f64(pool_in, kp + (size_t)t * d + i, elem_bytes);
                    vd[i] = elem_f64(pool_in, vp + (size_t)t * d + i, elem_bytes);
                }
                for (int g = 0; g < group; ++g) {
                    const double* q = qd + (size_t)g * d;
                    double* o = out + ((size_t)r * hq + j * group + g) * d;
                    double sc = 0.0;
                    for (int i = 0; i < d; ++i) sc += kd[i] * q[i];
                    sc *= scale;
                    if (sc > mx[g]) {
                        const double shrink = exp(mx[g] - sc);
                        den[g] *= shrink;
                        for (int i = 0; i < d; ++i) o[i] *= shrink;
                        mx[g] = sc;
                    }
                    const double wt = exp(sc - mx[g]);
                    den[g] += wt;
                    for (int i = 0; i < d; ++i) o[i] += wt * vd[i];
                }
            }
        }
        for (int g = 0; g < group; ++g) {
            const int h = j * group + g;
            double* o = out + ((size_t)r * hq + h) * d;
            if (ntok == 0) {  /* zero-token shard: O = 0, LSE = -inf (weight 0 in any merge) */
                lse[(size_t)r * hq + h] = -INFINITY;
                continue;
            }
            for (int i = 0; i < d; ++i) o[i] /= den[g];
            lse[(size_t)r * hq + h] = mx[g] + log(den[g]);
        }
        free(qd);
        free(kd);
        free(vd);
        free(mx);
        free(den);
    }
    return 0;
}

int dcpora_paged_decode_attn_f64(int nshards, int hq, int hkv, int d, int page_size,
                                 const uint16_t* q_bf16, const uint16_t* pool_bf16,
                                 const int32_t* block_table, const int32_t* cu_pages,
                                 const int64_t* shard_len, const uint8_t* page_fill, double scale,
                                 double* out, double* lse, int threads) {
    return dcpora_paged_decode_attn_any_f64(nshards, hq, hkv, d, page_size, 2, q_bf16, pool_bf16, block_table,
                                            cu_pages, shard_len, page_fill, scale, out, lse, threads);
}

/* MLA decode (K10).  The reference does not model MLA; this is
 * shard_attention<double> (attn_merge.hpp:53-82, same serial recurrence) with
 * keys = the dk-wide cache rows and values = their first dv columns, applied
 * per (shard, head) over a paged pool pool[frame][page_size][dk] (bf16 bits);
 * q is [nshards][heads][dk].  Zero-token shards give O = 0, LSE = -inf, as
 * dcp_mla_decode_attn does. */
int dcpora_shard_attention_kv_f64(const double* q, const double* k, const double* v, int64_t len, int dk,
                                  int dv, int v_stride, double scale, double* out, double* lse) {
    if (len < 1) return E_EMPTY; /* hpp:57 */
    double mx = -INFINITY, den = 0.0;
    for (int i = 0; i < dv; ++i) out[i] = 0.0;
    for (int64_t j = 0; j < len; ++j) {
        const double* kj = k + j * dk;
        const double* vj = v + j * v_stride;
        double s = 0.0;
        for (int i = 0; i < dk; ++i) s += kj[i] * q[i];
        s *= scale;
        if (s > mx) {
            const double shrink = exp(mx - s);
            den *= shrink;
            for (int i = 0; i < dv; ++i) out[i] *= shrink;
            mx = s;
        }
        const double w = exp(s - mx);
        den += w;
        for (int i = 0; i < dv; ++i) out[i] += w * vj[i];
    }
    for (int i = 0; i < dv; ++i) out[i] /= den;
    *lse = mx + log(den);
    return 0;
}

int dcpora_mla_paged_decode_f64(int nshards, int heads, int dk, int dv, int page_size, const uint16_t* q_bf16,
                                const uint16_t* pool_bf16, const int32_t* block_table, const int32_t* cu_pages,
                                const int64_t* shard_len, const uint8_t* page_fill, double scale, double* out,
                                double* lse, int threads) {
    int rc = 0;
    for (int r = 0; r < nshards; ++r) {
        const int p0 = cu_pages[r], p1 = cu_pages[r + 1];
        int64_t ntok = 0;
        for (int p = p0; p < p1; ++p) {
            const int64_t rem = shard_len[r] - (int64_t)(p - p0) * page_size;
            ntok += page_fill ? page_fill[p] : (rem < page_size ? rem : page_size);
        }
        if (ntok == 0) {
            for (int h = 0; h < heads; ++h) {
                for (int i = 0; i < dv; ++i) out[((size_t)r * heads + h) * dv + i] = 0.0;
                lse[(size_t)r * heads + h] = -INFINITY;
            }
            continue;
        }
        double* kd = malloc(sizeof(double) * (size_t)ntok * dk);
        int64_t t = 0;
        for (int p = p0; p < p1; ++p) {
            const int64_t rem = shard_len[r] - (int64_t)(p - p0) * page_size;
            const int fill = page_fill ? page_fill[p] : (int)(rem < page_size ? rem : page_size);
            const uint16_t* kp = pool_bf16 + (size_t)block_table[p] * page_size * dk;
            for (int s = 0; s < fill; ++s, ++t)
                for (int i = 0; i < dk; ++i) kd[(size_t)t * dk + i] = bf16_to_f64(kp[(size_t)s * dk + i]);
        }
#pragma omp parallel for schedule(dynamic) num_threads(threads > 0 ? threads : 1) reduction(min : rc)
        for (int h = 0; h < heads; ++h) {
            double qd[1024];
            for (int i = 0; i < dk; ++i) qd[i] = bf16_to_f64(q_bf16[((size_t)r * heads + h) * dk + i]);
            const int e = dcpora_shard_attention_kv_f64(qd, kd, kd, ntok, dk, dv, dk, scale,
                                                        out + ((size_t)r * heads + h) * dv, lse + (size_t)r * heads + h);
            rc = e < rc ? e : rc;
        }
        free(kd);
    }
    return rc;
}

/* ======================================================================
 * Planner — scheduler.cpp
 * ====================================================================== */

/* water_fill: scheduler.cpp:70-102.  Binary search for the minimal integer
 * level P with sum max(0, P-K_i) >= len over [0, max K + len]; split_i =
 * max(0, P-1-K_i); then one extra token, in participant order, to every
 * participant still below P until the remainder is exhausted. */
static void water_fill_impl(int n, int64_t len, const int64_t* K, int64_t* split) {
    int64_t lo = 0, hi = 0;
    for (int i = 0; i < n; ++i) hi = K[i] > hi ? K[i] : hi;
    hi += len;
    while (lo < hi) {
        const int64_t mid = lo + (hi - lo) / 2;
        int64_t cap = 0;
        for (int i = 0; i < n; ++i) cap += mid - K[i] > 0 ? mid - K[i] : 0;
        if (cap >= len) hi = mid; else lo = mid + 1;
    }
    int64_t assigned = 0;
    for (int i = 0; i < n; ++i) {
        const int64_t s = lo - 1 - K[i];
        split[i] = s > 0 ? s : 0;
        assigned += split[i];
    }
    int64_t rem = len - assigned;
    for (int i = 0; i < n && rem > 0; ++i)
        if (K[i] + split[i] < lo) { split[i] += 1; rem -= 1; }
}

int dcpora_water_fill(int n, const int32_t* participants, int64_t seq_len, const int64_t* loads,
                      int64_t* split) {
    (void)participants; /* used only for its size (scheduler.cpp:72) */
    water_fill_impl(n, seq_len, loads, split);
    return 0;
}

typedef struct {
    int64_t len[16];
    int deg[16];
    int n;
} Bucket;

static Bucket bucket_default(void) { /* scheduler.cpp:28-33 */
    Bucket b = {{32768, 131072, 393216, INT64_MAX}, {1, 2, 4, 8}, 4};
    return b;
}
static int bucket_lookup(const Bucket* b, int64_t len) { /* scheduler.cpp:10-14 */
    for (int i = 0; i < b->n; ++i)
        if (len <= b->len[i]) return b->deg[i];
    return b->deg[b->n - 1];
}
static int bucket_validate(const Bucket* b) { /* scheduler.cpp:16-26 */
    if (b->n == 0) return E_CONFIG;
    int64_t pl = 0;
    int pd = 0;
    for (int i = 0; i < b->n; ++i) {
        if (b->len[i] <= pl) return E_CONFIG;
        if (b->deg[i] < pd || b->deg[i] < 1) return E_CONFIG;
        pl = b->len[i];
        pd = b->deg[i];
    }
    return 0;
}
static int cp_degree_impl(int64_t len, const Bucket* b, int node_n) { /* scheduler.cpp:66-68 */
    const int d = bucket_lookup(b, len);
    return d < node_n ? d : node_n;
}

int dcpora_cp_degree(int64_t seq_len, const int64_t* bucket_len, const int* bucket_deg,
                     int n_bucket, int node_instances) {
    Bucket b = bucket_default();
    if (n_bucket > 0) {
        b.n = n_bucket;
        for (int i = 0; i < n_bucket; ++i) { b.len[i] = bucket_len[i]; b.deg[i] = bucket_deg[i]; }
    }
    return cp_degree_impl(seq_len, &b, node_instances);
}

/* ShapeSpace::default_space / bucket_shape: routing.cpp:89-109 (buckets in
 * lexicographic order; first componentwise-dominating one). */
int dcpora_bucket_shape_default(int m, int n, int* bm, int* bn) {
    static const int ms[] = {8, 16, 32, 64, 128, 256};
    static const int ns[] = {8, 16, 32, 64, 128, 256, 384, 512};
    if (m > 256 || n > 512) return E_SHAPE;
    for (int i = 0; i < 6; ++i)
        for (int j = 0; j < 8; ++j)
            if (ms[i] >= m && ns[j] >= n) { *bm = ms[i]; *bn = ns[j]; return 0; }
    *bm = 256;
    *bn = 512;
    return 0;
}

/* graph_memory_footprint: routing.cpp:111-127 on the default 48-bucket space. */
int dcpora_graph_footprint(int world, int heads, int head_size, int hidden, int max_blocks,
                           int elem, int idx, int64_t* graphs, int64_t* bytes) {
    const int64_t w = world, hn = heads, hs = head_size, mm = 256, nn = 512;
    const int64_t payload = (w * mm + w * nn) * hn * hs + w * nn * hs + mm * (int64_t)hidden;
    const int64_t index = mm * (int64_t)max_blocks + mm;
    *graphs = 48;
    *bytes = payload * elem + index * idx;
    return 0;
}

/* ---------------------------------------------------------------- world state */
#define MAXK 64

typedef struct {
    int32_t kv[MAXK];
    int64_t split[MAXK];
    int k;
    int32_t moe;
} Placement;

typedef struct {
    int64_t id, seq_len, generated;
    int state; /* 0 waiting, 1 active, 2 finished (types.hpp:32) */
    int has_p;
    Placement p;
} Req;

typedef struct {
    int32_t inst;
    int64_t frame;
} PageRef;

typedef struct {
    int64_t id;
    PageRef* pages;
    int64_t np, capp;
    int64_t trailing_fill, page_size;
    int64_t* shard_tokens; /* [W] */
} Entry;

typedef struct {
    int64_t kv_load, capacity, nfree;
    int moe_batch, shard_count, node;
    int64_t* free; /* LIFO, top at free[nfree-1] (page_table.hpp:19) */
} Inst;

typedef struct {
    int nodes, ipn, W;
    int64_t page, capacity;
    Inst* inst;
    Entry* ent; /* sorted by id (std::map order, page_table.hpp:96) */
    int64_t nent, capent;
    Req* req;
    int64_t nreq, capreq;
    int64_t* waiting;
    int64_t nwait, capwait;
    int kind, udeg, hol_strict;
    Bucket bucket;
    int* ucp_rr;
    int n_rr;
} World;

static void* grow(void* p, int64_t* cap, int64_t need, size_t elem) {
    if (need <= *cap) return p;
    int64_t c = *cap ? *cap : 16;
    while (c < need) c *= 2;
    *cap = c;
    return realloc(p, (size_t)c * elem);
}

/* make_cluster: page_table.cpp:133-148 — LIFO stacks seeded so that frames are
 * handed out in ascending order (highest id at the bottom). */
void* dcpora_world_create(int nodes, int inst_per_node, int64_t page_size, int64_t capacity,
                          int kind, const int64_t* bucket_len, const int* bucket_deg, int n_bucket,
                          int uniform_degree, int hol_strict) {
    World* w = calloc(1, sizeof(World));
    w->nodes = nodes;
    w->ipn = inst_per_node;
    w->W = nodes * inst_per_node;
    w->page = page_size;
    w->capacity = capacity;
    w->inst = calloc((size_t)w->W, sizeof(Inst));
    for (int s = 0; s < w->W; ++s) {
        Inst* in = &w->inst[s];
        in->node = s / inst_per_node;
        in->capacity = capacity;
        in->nfree = capacity;
        in->free = malloc(sizeof(int64_t) * (size_t)(capacity > 0 ? capacity : 1));
        for (int64_t f = 0; f < capacity; ++f) in->free[f] = capacity - 1 - f;
    }
    w->kind = kind;
    w->udeg = uniform_degree;
    w->hol_strict = hol_strict;
    w->bucket = bucket_default();
    if (n_bucket > 0) {
        w->bucket.n = n_bucket;
        for (int i = 0; i < n_bucket; ++i) { w->bucket.len[i] = bucket_len[i]; w->bucket.deg[i] = bucket_deg[i]; }
    }
    return w;
}

void dcpora_world_destroy(void* h) {
    World* w = h;
    if (!w) return;
    for (int s = 0; s < w->W; ++s) free(w->inst[s].free);
    for (int64_t i = 0; i < w->nent; ++i) { free(w->ent[i].pages); free(w->ent[i].shard_tokens); }
    free(w->inst);
    free(w->ent);
    free(w->req);
    free(w->waiting);
    free(w->ucp_rr);
    free(w);
}

int dcpora_world_enqueue(void* h, int64_t id, int64_t seq_len) {
    World* w = h;
    w->req = grow(w->req, &w->capreq, w->nreq + 1, sizeof(Req));
    Req* r = &w->req[w->nreq];
    memset(r, 0, sizeof(*r));
    r->id = id;
    r->seq_len = seq_len;
    w->waiting = grow(w->waiting, &w->capwait, w->nwait + 1, sizeof(int64_t));
    w->waiting[w->nwait++] = w->nreq++;
    return 0;
}

static int64_t ent_find(const World* w, int64_t id) { /* index or -(insert pos)-1 */
    int64_t lo = 0, hi = w->nent;
    while (lo < hi) {
        const int64_t mid = (lo + hi) / 2;
        if (w->ent[mid].id < id) lo = mid + 1; else hi = mid;
    }
    if (lo < w->nent && w->ent[lo].id == id) return lo;
    return -lo - 1;
}

/* GlobalPageTable::allocate: page_table.cpp:9-49 */
static int pt_allocate(World* w, const Req* r, const Placement* p) {
    int64_t pos = ent_find(w, r->id);
    if (pos >= 0) return E_FRAMES;        /* cpp:13-14 */
    if (r->seq_len < 1) return E_FRAMES;  /* cpp:15-16 */
    for (int i = 0; i < p->k; ++i) {      /* feasibility first, cpp:19-26 */
        const int64_t need = pages_for(p->split[i], w->page);
        if (w->inst[p->kv[i]].nfree < need) return E_FRAMES;
    }
    pos = -pos - 1;
    w->ent = grow(w->ent, &w->capent, w->nent + 1, sizeof(Entry));
    memmove(&w->ent[pos + 1], &w->ent[pos], sizeof(Entry) * (size_t)(w->nent - pos));
    w->nent++;
    Entry* e = &w->ent[pos];
    memset(e, 0, sizeof(*e));
    e->id = r->id;
    e->page_size = w->page;
    e->shard_tokens = calloc((size_t)w->W, sizeof(int64_t));
    for (int i = 0; i < p->k; ++i) { /* cpp:30-44 */
        const int s = p->kv[i];
        const int64_t need = pages_for(p->split[i], w->page);
        Inst* in = &w->inst[s];
        e->pages = grow(e->pages, &e->capp, e->np + need, sizeof(PageRef));
        for (int64_t q = 0; q < need; ++q) {
            e->pages[e->np].inst = s;
            e->pages[e->np].frame = in->free[in->nfree - 1];
            e->np++;
            in->nfree--;
        }
        in->kv_load += p->split[i];
        e->shard_tokens[s] += p->split[i];
        if (p->split[i] > 0) {
            const int64_t rem = p->split[i] % w->page;
            e->trailing_fill = rem == 0 ? w->page : rem;
        }
    }
    return 0;
}

/* GlobalPageTable::release: page_table.cpp:51-66 — frames pushed back in page order. */
static int pt_release(World* w, int64_t id) {
    const int64_t pos = ent_find(w, id);
    if (pos < 0) return E_UNKNOWN_REQ;
    Entry* e = &w->ent[pos];
    for (int64_t q = 0; q < e->np; ++q) {
        Inst* in = &w->inst[e->pages[q].inst];
        in->free[in->nfree++] = e->pages[q].frame;
    }
    for (int s = 0; s < w->W; ++s) w->inst[s].kv_load -= e->shard_tokens[s];
    free(e->pages);
    free(e->shard_tokens);
    memmove(&w->ent[pos], &w->ent[pos + 1], sizeof(Entry) * (size_t)(w->nent - pos - 1));
    w->nent--;
    return 0;
}

/* rebalance_active: scheduler.cpp:43-64.  Actives ordered by (cp_degree, id);
 * m_r = argmin over P_r of B (ties to the lowest instance id); B[m_r]++. */
static int cmp_kid(const void* a, const void* b, void* ctx) {
    const World* w = ctx;
    const Req* x = &w->req[*(const int64_t*)a];
    const Req* y = &w->req[*(const int64_t*)b];
    if (x->p.k != y->p.k) return x->p.k < y->p.k ? -1 : 1;
    return x->id < y->id ? -1 : (x->id > y->id);
}
/* small insertion/merge sort with context (qsort_r portability) */
static void sort_idx(int64_t* a, int64_t n, int (*cmp)(const void*, const void*, void*), void* ctx) {
    if (n < 2) return;
    int64_t* tmp = malloc(sizeof(int64_t) * (size_t)n);
    for (int64_t width = 1; width < n; width *= 2) {
        for (int64_t i = 0; i < n; i += 2 * width) {
            int64_t l = i, m = i + width < n ? i + width : n, r = i + 2 * width < n ? i + 2 * width : n;
            int64_t x = l, y = m, k = l;
            while (x < m && y < r) tmp[k++] = cmp(&a[y], &a[x], ctx) < 0 ? a[y++] : a[x++];
            while (x < m) tmp[k++] = a[x++];
            while (y < r) tmp[k++] = a[y++];
        }
        memcpy(a, tmp, sizeof(int64_t) * (size_t)n);
    }
    free(tmp);
}

static void rebalance(World* w) {
    for (int s = 0; s < w->W; ++s) w->inst[s].moe_batch = 0;
    int64_t n = 0;
    int64_t* act = malloc(sizeof(int64_t) * (size_t)(w->nreq + 1));
    for (int64_t i = 0; i < w->nreq; ++i)
        if (w->req[i].state == 1) act[n++] = i;
    sort_idx(act, n, cmp_kid, w);
    for (int64_t i = 0; i < n; ++i) {
        Placement* p = &w->req[act[i]].p;
        int32_t best = p->kv[0];
        for (int j = 0; j < p->k; ++j) {
            const int32_t s = p->kv[j];
            const int bs = w->inst[s].moe_batch, bb = w->inst[best].moe_batch;
            if (bs < bb || (bs == bb && s < best)) best = s;
        }
        p->moe = best;
        w->inst[best].moe_batch += 1;
    }
    free(act);
}

/* place_dcp: scheduler.cpp:130-170 (Alg. 1 lines 7-12). */
static void place_dcp(const World* w, const Req* r, Placement* p) {
    int best_node = 0;
    int64_t best_bn = INT64_MAX;
    for (int n = 0; n < w->nodes; ++n) { /* cpp:133-141 */
        int64_t bn = 0;
        for (int s = n * w->ipn; s < (n + 1) * w->ipn; ++s) bn += w->inst[s].moe_batch;
        if (bn < best_bn) { best_bn = bn; best_node = n; }
    }
    const int k = cp_degree_impl(r->seq_len, &w->bucket, w->ipn);
    const int nb = best_node * w->ipn, ne = nb + w->ipn;
    int moe = nb; /* min_batch_instance, cpp:118-126 */
    for (int s = nb; s < ne; ++s)
        if (w->inst[s].moe_batch < w->inst[moe].moe_batch) moe = s;
    /* SelectSmallestKV: node minus moe ordered by (K, id), cpp:148-156 */
    int32_t rest[MAXK];
    int nr = 0;
    for (int s = nb; s < ne; ++s)
        if (s != moe) rest[nr++] = s;
    for (int i = 1; i < nr; ++i) { /* insertion sort on a total order */
        const int32_t x = rest[i];
        int j = i - 1;
        while (j >= 0 && (w->inst[rest[j]].kv_load > w->inst[x].kv_load ||
                          (w->inst[rest[j]].kv_load == w->inst[x].kv_load && rest[j] > x))) {
            rest[j + 1] = rest[j];
            --j;
        }
        rest[j + 1] = x;
    }
    p->moe = moe;
    p->k = 0;
    p->kv[p->k++] = moe;
    for (int i = 0; i + 1 < k && i < nr; ++i) p->kv[p->k++] = rest[i];
    int64_t loads[MAXK];
    for (int i = 0; i < p->k; ++i) loads[i] = w->inst[p->kv[i]].kv_load;
    water_fill_impl(p->k, r->seq_len, loads, p->split);
}

/* place_single: scheduler.cpp:172-187 (LeastBatch / LeastCache). */
static void place_single(const World* w, const Req* r, Placement* p, int by_batch) {
    int best = 0;
    for (int s = 1; s < w->W; ++s) {
        const int better = by_batch ? w->inst[s].moe_batch < w->inst[best].moe_batch
                                    : w->inst[s].kv_load < w->inst[best].kv_load;
        if (better) best = s;
    }
    p->moe = best;
    p->k = 1;
    p->kv[0] = best;
    p->split[0] = r->seq_len;
}

/* place_uniform: scheduler.cpp:189-223 (Helix-style UniformCP). */
static void place_uniform(World* w, const Req* r, Placement* p) {
    const int d = w->udeg;
    const int total = (w->ipn / d) * w->nodes;
    if (w->n_rr != total) {
        free(w->ucp_rr);
        w->ucp_rr = calloc((size_t)total, sizeof(int));
        w->n_rr = total;
    }
    int bg = 0;
    int64_t best = INT64_MAX;
    for (int g = 0; g < total; ++g) {
        int64_t b = 0;
        for (int s = g * d; s < g * d + d; ++s) b += w->inst[s].moe_batch;
        if (b < best) { best = b; bg = g; }
    }
    const int gb = bg * d;
    p->k = d;
    const int64_t base = r->seq_len / d;
    int64_t rem = r->seq_len % d;
    for (int i = 0; i < d; ++i) {
        p->kv[i] = gb + i;
        p->split[i] = base + (rem > 0 ? 1 : 0);
        if (rem > 0) rem -= 1;
    }
    const int rr = w->ucp_rr[bg];
    p->moe = gb + rr;
    w->ucp_rr[bg] = (rr + 1) % d;
}

/* never_fits: scheduler.cpp:225-243 (uses the first instance's capacity). */
static int never_fits(const World* w, const Req* r) {
    const int64_t demand = pages_for(r->seq_len, w->page);
    const int64_t per = w->inst[0].capacity;
    int64_t reach;
    if (w->kind == 0) {
        const int k = cp_degree_impl(r->seq_len, &w->bucket, w->ipn);
        reach = per * k - (k - 1);
    } else if (w->kind == 3) {
        reach = per * w->udeg - (w->udeg - 1);
    } else {
        reach = per;
    }
    return demand > reach;
}

/* can_allocate: scheduler.cpp:104-113. */
static int can_allocate(const World* w, const Placement* p) {
    for (int i = 0; i < p->k; ++i)
        if (w->inst[p->kv[i]].nfree < pages_for(p->split[i], w->page)) return 0;
    return 1;
}

/* Scheduler::step: scheduler.cpp:245-306. */
int dcpora_world_step(void* h, int64_t* committed, int* n_committed, int64_t* deferred,
                      int* n_deferred, int64_t* unsched, int* n_unsched, int64_t* hol) {
    World* w = h;
    *n_committed = *n_deferred = *n_unsched = 0;
    *hol = 0;
    if (w->kind == 0) {
        if (bucket_validate(&w->bucket)) { /* policy validity is the caller's (SPEC) */ }
        rebalance(w); /* cpp:250-255 */
    } else {           /* cpp:256-261: B from sticky m_r */
        for (int s = 0; s < w->W; ++s) w->inst[s].moe_batch = 0;
        for (int64_t i = 0; i < w->nreq; ++i)
            if (w->req[i].state == 1) w->inst[w->req[i].p.moe].moe_batch += 1;
    }
    int head_recorded = 0;
    int64_t scan = 0;
    while (scan < w->nwait) {
        Req* r = &w->req[w->waiting[scan]];
        if (never_fits(w, r)) { /* cpp:270-274 */
            unsched[(*n_unsched)++] = r->id;
            memmove(&w->waiting[scan], &w->waiting[scan + 1], sizeof(int64_t) * (size_t)(w->nwait - scan - 1));
            w->nwait--;
            continue;
        }
        Placement p;
        memset(&p, 0, sizeof(p));
        switch (w->kind) {
            case 0: place_dcp(w, r, &p); break;
            case 1: place_single(w, r, &p, 1); break;
            case 2: place_single(w, r, &p, 0); break;
            default: place_uniform(w, r, &p); break;
        }
        if (can_allocate(w, &p)) { /* cpp:284-294 */
            r->p = p;
            r->has_p = 1;
            const int rc = pt_allocate(w, r, &p);
            if (rc) return rc;
            r->state = 1;
            w->inst[p.moe].moe_batch += 1;
            for (int i = 0; i < p.k; ++i) w->inst[p.kv[i]].shard_count += 1;
            committed[(*n_committed)++] = r->id;
            memmove(&w->waiting[scan], &w->waiting[scan + 1], sizeof(int64_t) * (size_t)(w->nwait - scan - 1));
            w->nwait--;
            continue;
        }
        deferred[(*n_deferred)++] = r->id; /* cpp:296-303 */
        if (scan == 0 && !head_recorded) {
            int64_t total_free = 0;
            for (int s = 0; s < w->W; ++s) total_free += w->inst[s].nfree;
            if (total_free >= pages_for(r->seq_len, w->page)) *hol += 1;
            head_recorded = 1;
        }
        if (w->hol_strict) break;
        ++scan;
    }
    return 0;
}

static Req* find_req(World* w, int64_t id) {
    for (int64_t i = 0; i < w->nreq; ++i)
        if (w->req[i].id == id) return &w->req[i];
    return NULL;
}

int dcpora_world_finish(void* h, int64_t id) {
    World* w = h;
    const int rc = pt_release(w, id);
    if (rc) return rc;
    Req* r = find_req(w, id);
    if (r) r->state = 2;
    return 0;
}

/* GlobalPageTable::append_token: page_table.cpp:86-121. */
int dcpora_world_append_token(void* h, int64_t id, int32_t* instance) {
    World* w = h;
    Req* r = find_req(w, id);
    if (!r || !r->has_p) return E_UNKNOWN_REQ;
    const int64_t pos = ent_find(w, id);
    if (pos < 0) return E_UNKNOWN_REQ;
    Entry* e = &w->ent[pos];
    if (e->np > 0 && e->trailing_fill < e->page_size) { /* cpp:93-99 */
        e->trailing_fill += 1;
        const int32_t t = e->pages[e->np - 1].inst;
        w->inst[t].kv_load += 1;
        e->shard_tokens[t] += 1;
        *instance = t;
        r->generated += 1;
        return 0;
    }
    int32_t t = e->np == 0 ? r->p.kv[0] : e->pages[e->np - 1].inst; /* cpp:101-103 */
    if (w->inst[t].nfree == 0) {
        t = -1;
        for (int i = 0; i < r->p.k; ++i)
            if (w->inst[r->p.kv[i]].nfree > 0) { t = r->p.kv[i]; break; }
        if (t < 0) { *instance = -1; return 0; } /* growth stall */
    }
    Inst* in = &w->inst[t];
    e->pages = grow(e->pages, &e->capp, e->np + 1, sizeof(PageRef));
    e->pages[e->np].inst = t;
    e->pages[e->np].frame = in->free[in->nfree - 1];
    e->np++;
    in->nfree--;
    e->trailing_fill = 1;
    in->kv_load += 1;
    e->shard_tokens[t] += 1;
    *instance = t;
    r->generated += 1;
    return 0;
}

int dcpora_world_placement(void* h, int64_t id, int32_t* kv, int64_t* split, int32_t* moe, int* k) {
    World* w = h;
    Req* r = find_req(w, id);
    if (!r || !r->has_p) return E_UNKNOWN_REQ;
    *k = r->p.k;
    *moe = r->p.moe;
    for (int i = 0; i < r->p.k; ++i) { kv[i] = r->p.kv[i]; split[i] = r->p.split[i]; }
    return 0;
}

int dcpora_world_instances(void* h, int64_t* kv_load, int32_t* moe_batch, int32_t* shard_count,
                           int64_t* free_frames) {
    World* w = h;
    for (int s = 0; s < w->W; ++s) {
        kv_load[s] = w->inst[s].kv_load;
        moe_batch[s] = w->inst[s].moe_batch;
        shard_count[s] = w->inst[s].shard_count;
        free_frames[s] = w->inst[s].nfree;
    }
    return w->W;
}

typedef struct {
    char* buf;
    int64_t cap, len;
} Sb;
static void sb_printf(Sb* s, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
#include <stdarg.h>
static void sb_printf(Sb* s, const char* fmt, ...) {
    char tmp[512];
    va_list ap;
    va_start(ap, fmt);
    const int n = vsnprintf(tmp, sizeof(tmp), fmt, ap);
    va_end(ap);
    if (s->buf && s->len + n < s->cap) memcpy(s->buf + s->len, tmp, (size_t)n + 1);
    s->len += n;
}

/* GlobalPageTable::dump_csv: page_table.cpp:123-131 (entries in id order). */
int dcpora_world_dump_page_table(void* h, char* buf, int64_t cap) {
    World* w = h;
    Sb s = {buf, cap, 0};
    if (buf && cap > 0) buf[0] = 0;
    sb_printf(&s, "request_id,logical_page,instance_id,frame_id\n");
    for (int64_t i = 0; i < w->nent; ++i)
        for (int64_t q = 0; q < w->ent[i].np; ++q)
            sb_printf(&s, "%lld,%lld,%d,%lld\n", (long long)w->ent[i].id, (long long)q,
                      w->ent[i].pages[q].inst, (long long)w->ent[i].pages[q].frame);
    return (int)s.len;
}

static int cmp_id(const void* a, const void* b, void* ctx) {
    const World* w = ctx;
    const int64_t x = w->req[*(const int64_t*)a].id, y = w->req[*(const int64_t*)b].id;
    return x < y ? -1 : (x > y);
}

/* build_binding_config + derive_routing_tables + dump_routing_csv:
 * routing.cpp:9-79.  Actives by id; M list at m_r with P_r; N list at every
 * s in P_r (zero-split members included, cpp:25-29) with m_r.  q_route is
 * N x W one-hot at m_r (cpp:40-49), res_route M x W ones at P_r (cpp:51-60). */
int dcpora_world_dump_routing(void* h, char* buf, int64_t cap) {
    World* w = h;
    int64_t n = 0;
    int64_t* act = malloc(sizeof(int64_t) * (size_t)(w->nreq + 1));
    for (int64_t i = 0; i < w->nreq; ++i)
        if (w->req[i].state == 1) act[n++] = i;
    sort_idx(act, n, cmp_id, w);
    for (int64_t i = 0; i < n; ++i) { /* cpp:19-21 */
        const Placement* p = &w->req[act[i]].p;
        int holds = 0;
        for (int j = 0; j < p->k; ++j) holds |= p->kv[j] == p->moe;
        if (!holds) { free(act); return E_INCONS; }
    }
    Sb s = {buf, cap, 0};
    if (buf && cap > 0) buf[0] = 0;
    sb_printf(&s, "instance,table,row,request_id,columns\n");
    char* bits = malloc((size_t)w->W + 1);
    for (int inst = 0; inst < w->W; ++inst) {
        int row = 0;
        for (int64_t i = 0; i < n; ++i) { /* q_route rows: requests with a shard here */
            const Req* r = &w->req[act[i]];
            for (int j = 0; j < r->p.k; ++j) {
                if (r->p.kv[j] != inst) continue;
                for (int c = 0; c < w->W; ++c) bits[c] = c == r->p.moe ? '1' : '0';
                bits[w->W] = 0;
                sb_printf(&s, "%d,q_route,%d,%lld,%s\n", inst, row++, (long long)r->id, bits);
            }
        }
        row = 0;
        for (int64_t i = 0; i < n; ++i) { /* res_route rows: requests MoE-bound here */
            const Req* r = &w->req[act[i]];
            if (r->p.moe != inst) continue;
            for (int c = 0; c < w->W; ++c) bits[c] = '0';
            for (int j = 0; j < r->p.k; ++j) bits[r->p.kv[j]] = '1';
            bits[w->W] = 0;
            sb_printf(&s, "%d,res_route,%d,%lld,%s\n", inst, row++, (long long)r->id, bits);
        }
    }
    free(bits);
    free(act);
    return (int)s.len;
}

int dcpora_world_instance_shards(void* h, int inst, int64_t* ids, int32_t* cu, int32_t* frames,
                                 int64_t* tokens, int cap_shards, int cap_frames) {
    World* w = h;
    int ns = 0, nf = 0;
    cu[0] = 0;
    for (int64_t i = 0; i < w->nent; ++i) {
        const Entry* e = &w->ent[i];
        int has = 0;
        for (int64_t q = 0; q < e->np; ++q) has |= e->pages[q].inst == inst;
        const Req* r = find_req(w, e->id);
        int member = 0;
        if (r && r->has_p)
            for (int j = 0; j < r->p.k; ++j) member |= r->p.kv[j] == inst;
        if (!has && !member) continue;
        if (ns >= cap_shards) return -8;
        ids[ns] = e->id;
        tokens[ns] = e->shard_tokens[inst];
        for (int64_t q = 0; q < e->np; ++q)
            if (e->pages[q].inst == inst) {
                if (nf >= cap_frames) return -8;
                frames[nf++] = (int32_t)e->pages[q].frame;
            }
        cu[++ns] = nf;
    }
    return ns;
}

/* mt19937_64 (the standard-specified engine) + uniform01 / uniform_int:
 * workload.hpp:18-26 (53-bit mantissa from the top bits; clamp to hi). */
typedef struct {
    uint64_t mt[312];
    int i;
} Mt64;
static void mt_seed(Mt64* m, uint64_t s) {
    m->mt[0] = s;
    for (int i = 1; i < 312; ++i)
        m->mt[i] = 6364136223846793005ULL * (m->mt[i - 1] ^ (m->mt[i - 1] >> 62)) + (uint64_t)i;
    m->i = 312;
}
static uint64_t mt_next(Mt64* m) {
    if (m->i >= 312) {
        for (int i = 0; i < 312; ++i) {
            const uint64_t x = (m->mt[i] & 0xFFFFFFFF80000000ULL) | (m->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t y = x >> 1;
            if (x & 1) y ^= 0xB5026F5AA96619E9ULL;
            m->mt[i] = m->mt[(i + 156) % 312] ^ y;
        }
        m->i = 0;
    }
    uint64_t y = m->mt[m->i++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}
void dcpora_uniform_int(uint64_t seed, int64_t lo, int64_t hi, int n, int64_t* out) {
    Mt64 m;
    mt_seed(&m, seed);
    for (int i = 0; i < n; ++i) {
        const double u = ldexp((double)(mt_next(&m) >> 11), -53);
        const double span = (double)(hi - lo + 1);
        int64_t v = lo + (int64_t)(u * span);
        out[i] = v > hi ? hi : v;
    }
}

/* MoE expert layer oracle (see dcp_oracle.h).  Experts are visited in
 * ascending id order; every product is fp64 over widened bf16 values. */
int dcpora_moe_layer_f64(int T, int H, int I, int E, int k, const uint16_t* x, const int32_t* idx,
                         const float* w, const uint16_t* w_gate, const uint16_t* w_up,
                         const uint16_t* w_down, double* out, int threads) {
    (void)E;
#pragma omp parallel for schedule(dynamic) num_threads(threads > 0 ? threads : 1)
    for (int t = 0; t < T; ++t) {
        double* o = out + (size_t)t * H;
        for (int h = 0; h < H; ++h) o[h] = 0.0;
        int order[64];
        for (int j = 0; j < k; ++j) order[j] = j;
        for (int a = 1; a < k; ++a) { /* ascending expert id */
            const int v = order[a];
            int b = a - 1;
            while (b >= 0 && idx[(size_t)t * k + order[b]] > idx[(size_t)t * k + v]) { order[b + 1] = order[b]; --b; }
            order[b + 1] = v;
        }
        double* act = malloc(sizeof(double) * (size_t)I);
        double* xd = malloc(sizeof(double) * (size_t)H);
        for (int h = 0; h < H; ++h) xd[h] = bf16_to_f64(x[(size_t)t * H + h]);
        for (int j = 0; j < k; ++j) {
            const int e = idx[(size_t)t * k + order[j]];
            const double we = (double)w[(size_t)t * k + order[j]];
            const uint16_t* g = w_gate + (size_t)e * I * H;
            const uint16_t* u = w_up + (size_t)e * I * H;
            const uint16_t* dn = w_down + (size_t)e * H * I;
            for (int i = 0; i < I; ++i) {
                double a = 0.0, b = 0.0;
                for (int h = 0; h < H; ++h) {
                    a += bf16_to_f64(g[(size_t)i * H + h]) * xd[h];
                    b += bf16_to_f64(u[(size_t)i * H + h]) * xd[h];
                }
                act[i] = a / (1.0 + exp(-a)) * b;
            }
            for (int h = 0; h < H; ++h) {
                double acc = 0.0;
                for (int i = 0; i < I; ++i) acc += bf16_to_f64(dn[(size_t)h * I + i]) * act[i];
                o[h] += we * acc;
            }
        }
        free(act);
        free(xd);
    }
    return 0;
}
