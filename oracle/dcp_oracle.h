/* SPDX-License-Identifier: Apache-2.0
 *
 * TEST INFRASTRUCTURE ONLY — the CPU restatement ("port") oracle.
 *
 * A plain-C restatement of the reference dcpsim algorithms on the DCP decode
 * path, used by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg as the checker.  The product (paper_2605_21100_b200/) never links or
 * calls it.  Every function cites the reference file:line it restates
 * (paths relative to /root/reference/proj).
 *
 * Parity pinning: tests/test_oracle.py checks this restatement against the
 * reference itself compiled from its own sources (oracle/_ref, see Makefile)
 * and against the SPEC known-answer vectors committed in tests/golden/.
 */
#ifndef DCP_ORACLE_H_
#define DCP_ORACLE_H_
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- attention (attn_merge.hpp / attn_merge.cpp) ---- */
int dcpora_shard_attention_f64(const double* q, const double* k, const double* v, int64_t len,
                               int d, double scale, double* out, double* lse);
int dcpora_shard_attention_f32(const float* q, const float* k, const float* v, int64_t len, int d,
                               float scale, float* out, float* lse);
int dcpora_reference_attention_f64(const double* q, const double* k, const double* v, int64_t len,
                                   int d, double scale, double* out);
int dcpora_lse_merge_f64(int n, const double* outs, const double* lses, int d, double* out);
int dcpora_sharded_attention_merge_f64(const double* q, const double* k, const double* v,
                                       int64_t len, int d, double scale, const int64_t* bounds,
                                       int nb, double* out);
int dcpora_sharded_attention_merge_f32(const float* q, const float* k, const float* v, int64_t len,
                                       int d, float scale, const int64_t* bounds, int nb,
                                       float* out);
/* Paged bf16 decode attention in fp64 over exactly-widened bf16 inputs; the
 * same argument meaning as dcp_splitkv_decode_attn (dcp_capi.h).  Zero-token
 * shards give out = 0, lse = -inf. */
int dcpora_paged_decode_attn_f64(int nshards, int hq, int hkv, int d, int page_size,
                                 const uint16_t* q_bf16, const uint16_t* pool_bf16,
                                 const int32_t* block_table, const int32_t* cu_pages,
                                 const int64_t* shard_len, const uint8_t* page_fill, double scale,
                                 double* out, double* lse, int threads);

/* ---- planner pieces (scheduler.cpp) ---- */
int dcpora_shard_attention_kv_f64(const double* q, const double* k, const double* v, int64_t len, int dk,
                                  int dv, int v_stride, double scale, double* out, double* lse);
int dcpora_mla_paged_decode_f64(int nshards, int heads, int dk, int dv, int page_size, const uint16_t* q_bf16,
                                const uint16_t* pool_bf16, const int32_t* block_table, const int32_t* cu_pages,
                                const int64_t* shard_len, const uint8_t* page_fill, double scale, double* out,
                                double* lse, int threads);
int dcpora_water_fill(int n, const int32_t* participants, int64_t seq_len, const int64_t* loads,
                      int64_t* split);
int dcpora_cp_degree(int64_t seq_len, const int64_t* bucket_len, const int* bucket_deg,
                     int n_bucket, int node_instances);
int dcpora_bucket_shape_default(int m, int n, int* bm, int* bn);
int dcpora_graph_footprint(int world, int heads, int head_size, int hidden, int max_blocks,
                           int elem, int idx, int64_t* graphs, int64_t* bytes);

/* ---- world: cluster + scheduler + requests (same surface as oracle/ref_shim.cpp) ---- */
void* dcpora_world_create(int nodes, int inst_per_node, int64_t page_size, int64_t capacity,
                          int kind, const int64_t* bucket_len, const int* bucket_deg, int n_bucket,
                          int uniform_degree, int hol_strict);
void dcpora_world_destroy(void* h);
int dcpora_world_enqueue(void* h, int64_t id, int64_t seq_len);
int dcpora_world_step(void* h, int64_t* committed, int* n_committed, int64_t* deferred,
                      int* n_deferred, int64_t* unsched, int* n_unsched, int64_t* hol);
int dcpora_world_finish(void* h, int64_t id);
int dcpora_world_append_token(void* h, int64_t id, int32_t* instance);
int dcpora_world_placement(void* h, int64_t id, int32_t* kv, int64_t* split, int32_t* moe, int* k);
int dcpora_world_instances(void* h, int64_t* kv_load, int32_t* moe_batch, int32_t* shard_count,
                           int64_t* free_frames);
int dcpora_world_dump_page_table(void* h, char* buf, int64_t cap);
int dcpora_world_dump_routing(void* h, char* buf, int64_t cap);
/* Per-shard page lists of instance `inst` for the Active requests, ordered by
 * request id: for each (request with a shard here) its frame ids in logical
 * order.  Returns number of shards; fills ids[], cu[] (n+1), frames[]. */
int dcpora_world_instance_shards(void* h, int inst, int64_t* ids, int32_t* cu, int32_t* frames,
                                 int64_t* tokens, int cap_shards, int cap_frames);

/* Same over bf16 (elem_bytes 2) or fp32 (elem_bytes 4) q / pool. */
int dcpora_paged_decode_attn_any_f64(int nshards, int hq, int hkv, int d, int page_size, int elem_bytes,
                                     const void* q, const void* pool, const int32_t* block_table,
                                     const int32_t* cu_pages, const int64_t* shard_len, const uint8_t* page_fill,
                                     double scale, double* out, double* lse, int threads);

/* MoE layer oracle (no reference implementation exists: parity unpinned vs the
 * reference; this restatement is the definition the device K4/K5 path is
 * checked against).  Per token t:
 *   out_t = sum over its top-k experts e in ascending id order of
 *           w_{t,e} * W_down_e( silu(W_gate_e x_t) * (W_up_e x_t) )
 * in fp64 over exactly-widened bf16 inputs.  w_gate/w_up: [E][I][H],
 * w_down: [E][H][I] (bf16 bits), x: [T][H], idx/w: [T][k]. */
int dcpora_moe_layer_f64(int T, int H, int I, int E, int k, const uint16_t* x, const int32_t* idx,
                         const float* w, const uint16_t* w_gate, const uint16_t* w_up,
                         const uint16_t* w_down, double* out, int threads);

void dcpora_uniform_int(uint64_t seed, int64_t lo, int64_t hi, int n, int64_t* out);

#ifdef __cplusplus
}
#endif
#endif
