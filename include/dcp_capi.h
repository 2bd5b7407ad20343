/* SPDX-License-Identifier: Apache-2.0
 *
 * dcp_capi.h — C ABI of the B200-native DCP decode-step data path.
 *
 * The reference (`/root/reference/proj`, namespace dcpsim) is a header-level
 * C++20 library with no C ABI and no device code.  This header is the thin
 * layer a caller (the dcpsim C++ drop-in in include/dcpsim/, ctypes tests,
 * cgo / JNI bindings) binds to reach the sm_100a kernels.  Each entry point
 * names the reference interface whose semantics it implements.
 *
 * Conventions
 *   - Plain pointers and sizes only; no torch / C++ types.
 *   - Device pointers are caller-owned; no allocation inside hot calls.
 *   - Every call is stream-ordered on the `stream` argument (a cudaStream_t,
 *     passed as void* so this header needs no CUDA include); NULL = legacy
 *     default stream.
 *   - Return 0 on success or a negative DCP_E_* code.  One code per
 *     reference exception class (types.hpp:19-30) plus CUDA failures.
 *     `dcp_last_error()` returns a thread-local message for the last failure.
 *   - One host thread per dcp_ctx (mirrors the single-writer model,
 *     SPEC.md:98).
 */
#ifndef DCP_CAPI_H_
#define DCP_CAPI_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define DCP_API __attribute__((visibility("default")))
#else
#define DCP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: one per dcpsim exception (types.hpp:19-30) ---------- */
enum {
    DCP_OK = 0,
    DCP_E_INSUFFICIENT_FRAMES = -1,  /* dcpsim::InsufficientFrames   */
    DCP_E_UNKNOWN_REQUEST = -2,      /* dcpsim::UnknownRequest       */
    DCP_E_UNKNOWN_PAGE = -3,         /* dcpsim::UnknownPage          */
    DCP_E_INCONSISTENT = -4,         /* dcpsim::InconsistentPlacement */
    DCP_E_SHAPE_OVERFLOW = -5,       /* dcpsim::ShapeOverflow        */
    DCP_E_EMPTY_SHARD = -6,          /* dcpsim::EmptyShard           */
    DCP_E_CONFIG = -7,               /* dcpsim::ConfigError          */
    DCP_E_INVALID_ARG = -8,          /* bad pointer / size at the ABI */
    DCP_E_UNSUPPORTED = -9,          /* shape not compiled in         */
    DCP_E_CUDA = -10,                /* CUDA runtime / driver failure  */
    DCP_E_TIMEOUT = -11              /* an exchange flag wait timed out (peer lost / out of step) */
};

DCP_API const char* dcp_last_error(void);
DCP_API const char* dcp_version(void);

/* ---- context --------------------------------------------------------------- */
typedef struct dcp_ctx dcp_ctx;

/* Binds to CUDA device `device` (must be sm_100).  Caches the SM count and
 * TMA descriptors of registered KV pools. */
DCP_API int dcp_ctx_create(int device, dcp_ctx** out);
DCP_API int dcp_ctx_destroy(dcp_ctx* ctx);
DCP_API int dcp_ctx_num_sms(const dcp_ctx* ctx);
/* Measurement helper: a one-thread kernel that sleeps ~`microseconds` on the
 * stream, so a host can enqueue a whole step behind it and per-kernel events
 * then time device work only (no host launch gaps). */
DCP_API int dcp_device_sleep(dcp_ctx* ctx, int32_t microseconds, void* stream);
/* Synchronous device->host copy of `bytes` (for hosts that bind only this ABI). */
DCP_API int dcp_copy_to_host(void* dst, const void* src, size_t bytes);

/* ---- K1 + K9: split-KV paged decode attention --------------------------------
 *
 * Implements, per (shard, q-head), the semantics of
 *   dcpsim::shard_attention<T>   attn_merge.hpp:53-82   (partial O + natural-log LSE)
 * over the paged KV a GlobalPageTable lays out (page_table.cpp:9-49), and the
 * intra-GPU split combine with the math of
 *   dcpsim::lse_merge<T>         attn_merge.hpp:86-100.
 * A "shard" is one (request, instance) KV shard; for single-GPU decode each
 * request is one shard.
 *
 * Paged KV pool (bf16), one frame per page:
 *   pool[frame][kv ∈ {K,V}][kv_head][page_size][head_dim]
 * Shard r owns pages block_table[cu_pages[r] .. cu_pages[r+1]) (frame ids, in
 * logical order) and shard_len[r] tokens; page j of the shard holds
 * page_fill[cu_pages[r]+j] valid tokens (1..page_size) when page_fill is
 * non-NULL, else min(page_size, shard_len - j*page_size).
 * Zero-token shards are accepted (routing tables include them,
 * routing.cpp:25-29): their LSE is -inf and O is 0 (weight 0 in any merge),
 * where dcpsim::shard_attention would throw EmptyShard (hpp:57).
 *
 * q:   bf16 [num_shards][num_q_heads][head_dim]
 * out: fp32 [num_shards][num_q_heads][head_dim]   softmax-normalised over the shard
 * lse: fp32 [num_shards][num_q_heads]             natural log, as hpp:80
 * Compiled shapes: head_dim 128, page_size 16 / 32 / 64, (num_kv_heads, group) in
 * {(8,4), (4,8), (8,1), (2,16), (1,16)}.  Other shapes return DCP_E_UNSUPPORTED.
 *
 * workspace: device buffer of dcp_attn_workspace_bytes(...) bytes, zeroed once
 * before first use (cudaMemset); the kernel leaves it zeroed again. */
typedef struct dcp_attn_args {
    int32_t num_shards;
    int32_t num_q_heads;
    int32_t num_kv_heads;
    int32_t head_dim;
    int32_t page_size;
    int64_t num_frames;         /* frames in the pool */
    const void* q;              /* bf16 */
    const void* kv_pool;        /* bf16, 16-byte aligned */
    const int32_t* block_table; /* [cu_pages[num_shards]] frame ids */
    const int32_t* cu_pages;    /* [num_shards+1], cu_pages[0] == 0 */
    const int64_t* shard_len;   /* [num_shards] tokens */
    const uint8_t* page_fill;   /* optional [cu_pages[num_shards]] */
    float scale;                /* softmax scale, 1/sqrt(head_dim) by convention */
    float* out;
    float* lse;
    void* workspace;
    size_t workspace_bytes;
} dcp_attn_args;

DCP_API size_t dcp_attn_workspace_bytes(const dcp_ctx* ctx, int32_t num_shards, int32_t num_q_heads,
                                int32_t head_dim);
DCP_API int dcp_splitkv_decode_attn(dcp_ctx* ctx, const dcp_attn_args* args, void* stream);

/* K1-f32: the same call in fp32 — the reference's production precision
 * (shard_attention<float> / lse_merge<float>, attn_merge.cpp:64-77; SPEC.md:380
 * rel <= 1e-5).  q fp32 [num_shards][num_q_heads][128], kv_pool fp32
 * [frames][2][num_kv_heads][page_size][128] (16-byte aligned); any page_size
 * 1..255; num_kv_heads <= 8, group in {1, 2, 4, 8}.  CUDA-core fp32 FMAs and
 * expf / logf throughout (no reduced-precision step).  Same workspace. */
DCP_API int dcp_splitkv_decode_attn_f32(dcp_ctx* ctx, const dcp_attn_args* args, void* stream);

/* Number of kernel launches the last dcp_splitkv_decode_attn issued (for the
 * bench's gpu_launches accounting). */
DCP_API int dcp_attn_launches_per_call(void);
/* Debug: per-CTA globaltimer stamps of later K1 launches into a device buffer of
 * num_sms x 8 int64 (NULL = off): entry, first ring stage, last segment end, ticket,
 * merge end, exit, SM id, pages. */
DCP_API int dcp_k1_set_trace(void* dev_buf);

/* ---- K10: MLA split-KV paged decode attention (tcgen05, CTA pairs) ------------
 *
 * The DeepSeek-V3 absorbed-latent decode shape of cfg5.  Per
 * (shard, q-head) the semantics are dcpsim::shard_attention<T>
 * (attn_merge.hpp:53-82) with keys = the 576-wide cache rows (kv_lora_rank 512
 * latent | 64 rope) and values = their first 512 columns; the intra-GPU split
 * combine is lse_merge (hpp:86-100).  The reference does not model MLA
 * (SPEC.md:381); the shard / page / fill conventions are those of
 * dcp_splitkv_decode_attn above.
 *
 * q:       bf16 [num_shards][128][576]  (absorbed q_nope | q_pe)
 * kv_pool: bf16 [num_frames][page_size][576]  (c_kv | k_pe), 16-byte aligned
 * out:     fp32 [num_shards][128][512]  softmax-normalised over the shard
 * lse:     fp32 [num_shards][128]       natural log
 * Compiled: num_q_heads 128, kv_lora_rank 512, rope_dim 64, page_size 16/32/64.
 * workspace: dcp_mla_workspace_bytes(...) bytes (no zeroing needed); each call
 * issues 3 kernels (tile scan, the CTA-pair kernel, the split merge). */
typedef struct dcp_mla_args {
    int32_t num_shards;
    int32_t num_q_heads;
    int32_t kv_lora_rank;
    int32_t rope_dim;
    int32_t page_size;
    int64_t num_frames;
    const void* q;
    const void* kv_pool;
    const int32_t* block_table;
    const int32_t* cu_pages;
    const int64_t* shard_len;
    const uint8_t* page_fill;   /* optional */
    float scale;                /* softmax scale (DeepSeek-V3: 1/sqrt(192) x yarn mscale^2) */
    float* out;
    float* lse;
    void* workspace;
    size_t workspace_bytes;
} dcp_mla_args;

DCP_API size_t dcp_mla_workspace_bytes(const dcp_ctx* ctx, int32_t num_shards);
DCP_API int dcp_mla_decode_attn(dcp_ctx* ctx, const dcp_mla_args* args, void* stream);
DCP_API int dcp_mla_launches_per_call(void);

/* Diagnostics: record globaltimer stamps into a device buffer of 2048 + 3 x 256
 * int64: [0, 2048) = 256 x 8 for CTA pair 0 (per tile: MMA before-QK, after-QK,
 * after-P wait, after-PV; softmax S-ready / P-published for CTA 0 and CTA 1),
 * then per pair (start, end, SM id).  NULL switches it off. */
DCP_API int dcp_mla_set_trace(void* dev_buf);


/* ---- K6 + K7: the DCP planner on the device ----------------------------------
 *
 * Device-resident cluster state (InstanceState K_s/B_s/R_i + LIFO free-frame
 * stacks, page_table.hpp:13-25, make_cluster page_table.cpp:133-148), the
 * global page table (page_table.hpp:36-74) and the FIFO waiting queue.
 * Semantics are the reference's, bit-exact:
 *   dcp_planner_step         Scheduler::step             scheduler.cpp:245-306
 *                            (rebalance_active, place_dcp / place_single /
 *                            place_uniform, water_fill, can_allocate,
 *                            never_fits, GlobalPageTable::allocate)
 *   dcp_planner_finish       pt_free / GlobalPageTable::release  page_table.cpp:51-66
 *   dcp_planner_append_token GlobalPageTable::append_token       page_table.cpp:86-121
 *   dcp_planner_build_routing build_binding_config + derive_routing_tables
 *                            + bucket_shape              routing.cpp:9-63, 101-109
 *   dcp_planner_dump_*       GlobalPageTable::dump_csv / dump_routing_csv
 *                                                        page_table.cpp:123-131, routing.cpp:65-79
 * The active set of a step is every request committed and not yet finished
 * (the `active` span of Scheduler::step).  Limits: world size <= 32,
 * instances_per_node <= 16, capacity_pages < 2^31.
 * Errors: InsufficientFrames(-1) for a zero-length request reaching
 * allocate, UnknownRequest(-2) for finish/append of an unknown id,
 * ConfigError(-7) for an invalid policy (SchedulerPolicy::validate,
 * scheduler.cpp:35-41), InconsistentPlacement(-4) from build_routing. */
typedef struct dcp_planner dcp_planner;

enum { DCP_POLICY_DCP = 0, DCP_POLICY_LEAST_BATCH = 1, DCP_POLICY_LEAST_CACHE = 2,
       DCP_POLICY_UNIFORM_CP = 3 };

typedef struct dcp_planner_config {
    int32_t nodes;
    int32_t instances_per_node;
    int64_t page_size;
    int64_t capacity_pages;     /* per instance */
    int32_t policy;             /* DCP_POLICY_* (PolicyKind, scheduler.hpp:29) */
    int32_t n_bucket;           /* 0 = BucketFn::default_table() */
    const int64_t* bucket_len;  /* host, inclusive upper bounds */
    const int32_t* bucket_deg;  /* host */
    int32_t uniform_degree;
    int32_t hol_strict;
    int32_t max_requests;       /* concurrent request slots */
    int64_t reserve_pages;      /* per-request page-list growth reserve */
} dcp_planner_config;

/* Read-only device view of one instance after dcp_planner_build_routing:
 * the K1 inputs of that instance (shards = its N list, in request-id order). */
typedef struct dcp_instance_view {
    int32_t n_rows;             /* N: shards held here */
    int32_t m_rows;             /* M: requests MoE-bound here */
    int32_t bucket_m, bucket_n; /* bucket_shape(M, N); -1 on ShapeOverflow */
    const int64_t* n_ids;       /* [N] */
    const int32_t* n_moe;       /* [N] m_r of each shard request */
    const uint8_t* q_route;     /* [N][W] */
    const int64_t* m_ids;       /* [M] */
    const uint8_t* res_route;   /* [M][W] */
    const int32_t* cu_pages;    /* [N+1] */
    const int64_t* shard_len;   /* [N] */
    const int32_t* block_table; /* [cu_pages[N]] */
    const uint8_t* page_fill;   /* [cu_pages[N]] */
    /* exchange maps for the routed step (dcp_route_q / dcp_decode_attn_routed / dcp_merge_partials) */
    const int32_t* n_mrow;      /* [N] row of each shard's request in m_r's M list */
    const int32_t* m_nrow;      /* [M][W] row of each M request in s' N list (-1: s' not in P_r) */
    const int32_t* m_k;         /* [M] |P_r| */
    const int32_t* m_kv;        /* [M][16] P_r in kv_binding order */
    const int32_t* m_count_all; /* [W] device copy of every instance's M */
    const int32_t* n_count_dev; /* device copy of this instance's N */
    int32_t world;
    int32_t instance;
    const int32_t* total_pages_dev; /* device copy of cu_pages[N] (K1 reads it with N, not after it) */
} dcp_instance_view;

DCP_API int dcp_planner_create(dcp_ctx* ctx, const dcp_planner_config* cfg, dcp_planner** out);
DCP_API int dcp_planner_destroy(dcp_planner* pl);
/* FIFO append (host arrays). */
DCP_API int dcp_planner_enqueue(dcp_planner* pl, const int64_t* ids, const int64_t* seq_lens,
                                int32_t n);
/* One scheduling round (K6), stream-ordered. */
DCP_API int dcp_planner_step(dcp_planner* pl, void* stream);
/* Synchronizes and copies the last StepResult out (host arrays sized >= queued count). */
DCP_API int dcp_planner_step_result(dcp_planner* pl, int64_t* committed, int32_t* n_committed,
                                    int64_t* deferred, int32_t* n_deferred, int64_t* unschedulable,
                                    int32_t* n_unschedulable, int64_t* hol_events);
DCP_API int dcp_planner_finish(dcp_planner* pl, const int64_t* ids, int32_t n, void* stream);
DCP_API int dcp_planner_append_token(dcp_planner* pl, const int64_t* ids, int32_t n,
                                     int32_t* out_instance);
DCP_API int dcp_planner_placement(dcp_planner* pl, int64_t id, int32_t* kv_binding, int64_t* split,
                                  int32_t* moe_binding, int32_t* cp_degree);
DCP_API int dcp_planner_instances(dcp_planner* pl, int64_t* kv_load, int32_t* moe_batch,
                                  int32_t* shard_count, int64_t* free_frames);
/* CSV writers; return the full length (write at most cap-1 bytes + NUL). */
DCP_API int64_t dcp_planner_dump_page_table(dcp_planner* pl, char* buf, int64_t cap);
DCP_API int dcp_planner_build_routing(dcp_planner* pl, void* stream);
DCP_API int64_t dcp_planner_dump_routing(dcp_planner* pl, char* buf, int64_t cap);
DCP_API int dcp_planner_instance_view(dcp_planner* pl, int32_t instance, dcp_instance_view* out);
/* Kernel launches issued by the last step / build_routing call. */
DCP_API int dcp_planner_last_launches(const dcp_planner* pl);

/* ---- K2 / K1-routed / K3: the routing-based exchange of one DCP step ---------
 *
 * The paper's backend: the sender reads the routing mask
 * and stores the payload directly into the peer's pre-allocated receive slot
 * (NVLink P2P when the peer is another GPU), the receiver polls an arrival
 * flag.  Phases (Fig. 7): 1 Q-route (dcp_route_q), 2 partial attention with
 * the Res-route put fused into its epilogue (dcp_decode_attn_routed), 4 LSE
 * merge at the MoE binding (dcp_merge_partials; math of lse_merge,
 * attn_merge.hpp:86-100, in kv_binding order, zero-token shards weight 0).
 * Pools per instance (one allocation, exported by CUDA IPC for peers), each
 * buffer twice (selected by the step epoch's parity):
 *   q_recv [n_max][HQ][q_dim] (bf16 or fp32) + flags,
 *   res [m_max][W][HQ][o_dim] fp32 + LSE [m_max][W][HQ] + flags, and a "done" word.
 * Local buffers: q_local [m_max][HQ][q_dim] (queries of the requests MoE-bound
 * here, in M-row order), out [m_max][HQ][o_dim] fp32 + out_lse.
 * Step protocol: flags carry a per-step epoch, so graph replay needs no reset.
 * All instances call dcp_xchg_begin_step once per step; it waits (on the
 * device) until every peer has begun the previous step, so no instance runs
 * more than one step ahead and the parity buffers are never overwritten while
 * a peer still reads them.  Every flag wait is bounded by timeout_ms: a lost or
 * mis-epoched flag leaves an error in the instance (kernels still terminate)
 * that dcp_xchg_status reports as DCP_E_TIMEOUT.
 * Widths: bf16 GQA/MHA (q_dim = o_dim = head_dim, q_elem_bytes 2), fp32
 * (q_elem_bytes 4, dcp_decode_attn_routed_f32), MLA (q_dim 576, o_dim 512,
 * dcp_mla_decode_attn_routed).  hq * q_dim * q_elem_bytes must be a multiple
 * of 16 and o_dim a multiple of 32. */
typedef struct dcp_xchg dcp_xchg;
typedef struct dcp_xchg_config {
    int32_t world;
    int32_t self;
    int32_t num_q_heads;
    int32_t head_dim;
    int32_t n_max;        /* ShapeSpace n_max (routing.hpp:62-63) */
    int32_t m_max;        /* ShapeSpace m_max */
    int32_t q_dim;        /* Q width per head; 0 = head_dim */
    int32_t o_dim;        /* partial-O width per head; 0 = head_dim */
    int32_t q_elem_bytes; /* 2 (bf16) or 4 (fp32); 0 = 2 */
    int32_t timeout_ms;   /* flag-wait bound; 0 = 10000 */
} dcp_xchg_config;

DCP_API int dcp_xchg_create(dcp_ctx* ctx, const dcp_xchg_config* cfg, dcp_xchg** out);
DCP_API int dcp_xchg_destroy(dcp_xchg* x);
DCP_API int dcp_xchg_ipc_handle(dcp_xchg* x, void* handle64);
DCP_API int dcp_xchg_open_peer_ipc(dcp_xchg* x, int32_t peer, const void* handle64);
DCP_API int dcp_xchg_set_peer_local(dcp_xchg* x, int32_t peer, const dcp_xchg* other);
DCP_API int dcp_xchg_commit(dcp_xchg* x);
DCP_API int dcp_xchg_begin_step(dcp_xchg* x, void* stream);
DCP_API int dcp_xchg_buffers(dcp_xchg* x, void** q_local, void** q_recv, float** out,
                             float** out_lse);
/* Stage the queries of this instance's M requests (device bf16 [rows][HQ][D],
 * M-row order) into q_local (the output of the query projection in a model). */
DCP_API int dcp_xchg_write_queries(dcp_xchg* x, const void* q_rows, int32_t rows, void* stream);
DCP_API int dcp_route_q(dcp_xchg* x, const dcp_instance_view* v, void* stream);
/* K1 over this instance's N list (q from q_recv, waits on Q-route flags),
 * outputs stored into each row's m_r result slot.  `a` supplies kv_pool,
 * num_frames, head counts, scale and workspace (sized for n_max shards); its
 * q/out/lse/shard arrays are ignored. */
DCP_API int dcp_decode_attn_routed(dcp_ctx* ctx, dcp_xchg* x, const dcp_instance_view* v,
                                   const dcp_attn_args* a, void* stream);
/* K1-f32 routed: the fp32 variant of dcp_decode_attn_routed over an exchange
 * created with q_elem_bytes 4 (fp32 Q rows); kv_pool fp32 as dcp_splitkv_decode_attn_f32. */
DCP_API int dcp_decode_attn_routed_f32(dcp_ctx* ctx, dcp_xchg* x, const dcp_instance_view* v,
                                       const dcp_attn_args* a, void* stream);
/* K10 routed: the MLA decode of this instance's N list inside a DCP step (Fig. 7 phase 2
 * for cfg5).  The exchange must be MLA-shaped (num_q_heads 128, q_dim 576, o_dim 512,
 * q_elem_bytes 2): Q rows come from the receive pool after each row's Q-route flag, O and
 * LSE are stored into m_r's result slot and its flag published (Res-route put), so
 * dcp_route_q before and dcp_merge_partials after complete the step.  `a` supplies
 * kv_pool, num_frames, page_size, scale and a workspace of
 * dcp_mla_workspace_bytes(ctx, n_max) bytes; its q / shard arrays / out / lse are ignored.
 * Four launches (tile scan, ticket reset, the CTA-pair kernel, merge + flag publish). */
DCP_API int dcp_mla_decode_attn_routed(dcp_ctx* ctx, dcp_xchg* x, const dcp_instance_view* v,
                                       const dcp_mla_args* a, void* stream);
DCP_API int dcp_merge_partials(dcp_xchg* x, const dcp_instance_view* v, void* stream);
/* The whole routed step of one instance in ONE launch (Fig. 7 phases 1-4): the step fence
 * and epoch bump of dcp_xchg_begin_step, K2's Q-route puts in K1's prologue (while the
 * producer warp already streams KV), K1 + Res-route, and K3's LSE merges of this instance's
 * M rows in K1's epilogue — outputs where dcp_merge_partials puts them.  Equivalent to
 * begin_step + route_q + decode_attn_routed + merge_partials, bit for bit.  The epilogue
 * waits for the peers' partials inside the kernel, so every instance must be able to run
 * concurrently: one instance per GPU (or per process), or W = 1.  Instances sharing one GPU
 * in one process use the four phased calls instead. */
DCP_API int dcp_decode_step_fused(dcp_ctx* ctx, dcp_xchg* x, const dcp_instance_view* v,
                                  const dcp_attn_args* args, void* stream);
/* Synchronizes the device and reports the exchange error word: DCP_OK, or
 * DCP_E_TIMEOUT with info[0..3] = {code, where (site << 24 | peer << 16 | row),
 * wanted flag value, last value seen}; the word is cleared.  info may be NULL. */
DCP_API int dcp_xchg_status(dcp_xchg* x, uint32_t* info);

/* ---- entry points backing the dcpsim C++ drop-in (include/dcpsim/) ---------- */
/* Replace the active policy (SchedulerPolicy, scheduler.hpp:31-39).  The
 * UniformCP round-robin counters reset when the group count changes, as
 * ucp_round_robin_.assign does (scheduler.cpp:195-196). */
DCP_API int dcp_planner_set_policy(dcp_planner* pl, int32_t policy, int32_t n_bucket,
                                   const int64_t* bucket_len, const int32_t* bucket_deg,
                                   int32_t uniform_degree, int32_t hol_strict);
/* UniformCP round-robin counters (Scheduler::ucp_round_robin_, scheduler.hpp:88):
 * dir 0 uploads rr[0..n) (resizing the device vector), dir 1 reads them back.  The
 * C++ drop-in keeps them per Scheduler and pushes / pulls them around each step. */
DCP_API int dcp_planner_ucp_rr(dcp_planner* pl, int32_t* rr, int32_t n, int32_t dir);
/* Make the device waiting queue exactly `ids` (FIFO order).  Unknown ids are
 * admitted as new waiting requests with seq_lens[i]; known ids must be waiting.
 * Waiting requests not listed are dropped. */
DCP_API int dcp_planner_set_queue(dcp_planner* pl, const int64_t* ids, const int64_t* seq_lens,
                                  int32_t n);
/* GlobalPageTable::allocate with a caller-supplied placement
 * (page_table.cpp:9-49): InsufficientFrames(-1) leaves no partial state. */
DCP_API int dcp_planner_allocate(dcp_planner* pl, int64_t id, int64_t seq_len, int32_t cp_degree,
                                 const int32_t* kv_binding, const int64_t* split, int32_t moe_binding);
/* Page list of one tracked request (logical order); returns the page count. */
DCP_API int64_t dcp_planner_pages(dcp_planner* pl, int64_t id, int32_t* instance, int32_t* frame,
                                  int64_t cap);
/* moe_binding of every active request (ids and bindings, any order); returns count. */
DCP_API int32_t dcp_planner_active_moe(dcp_planner* pl, int64_t* ids, int32_t* moe, int32_t cap);
/* rebalance_active over an explicit active list (scheduler.cpp:43-64). */
DCP_API int dcp_planner_rebalance(dcp_planner* pl, const int64_t* ids, int32_t n);
/* Upload host instance state (kv_load, moe_batch, shard_count, LIFO stacks:
 * stacks[s*capacity .. + nfree[s]), bottom first) into an idle planner. */
DCP_API int dcp_planner_load_instances(dcp_planner* pl, const int64_t* kv_load,
                                       const int32_t* moe_batch, const int32_t* shard_count,
                                       const int64_t* nfree, const int32_t* stacks);
/* water_fill (scheduler.cpp:70-102) on the device; n <= 32 participants. */
DCP_API int dcp_water_fill(dcp_ctx* ctx, int32_t n, const int64_t* kv_loads, int64_t seq_len,
                           int64_t* split);
/* build_binding_config (routing.cpp:9-32) on the device for explicit placements
 * (host arrays; kv_binding flattened [n][16]).  Per instance s, n_rows[s*n ..]
 * and m_rows[s*n ..] receive the input indices of its N and M lists (id order). */
DCP_API int dcp_binding_config(dcp_ctx* ctx, int32_t n, const int64_t* ids, const int32_t* cp_degree,
                               const int32_t* moe_binding, const int32_t* kv_binding, int32_t world,
                               int32_t* n_count, int32_t* m_count, int32_t* n_rows, int32_t* m_rows);
/* derive_routing_tables (routing.cpp:34-63) expansion on the device: q bits
 * one-hot at shard_moe[r]; res bits at the set bits of res_mask[r]. */
DCP_API int dcp_route_tables(dcp_ctx* ctx, int32_t world, int32_t n_rows, const int32_t* shard_moe,
                             int32_t m_rows, const uint32_t* res_mask, uint8_t* q_bits,
                             uint8_t* res_bits);
/* shard_attention<T> (attn_merge.hpp:53-82) for a batch of items on the
 * device; dtype_bytes 4 (float) or 8 (double); device pointers. */
DCP_API int dcp_shard_attention_batch(dcp_ctx* ctx, int32_t dtype_bytes, int32_t n_items,
                                      int32_t head_dim, double scale, const void* q,
                                      const void* keys, const void* values, const int64_t* q_off,
                                      const int64_t* kv_off, const int64_t* len, void* out,
                                      void* lse, void* stream);
/* lse_merge<T> (attn_merge.hpp:86-100) per group of partials; device pointers. */
DCP_API int dcp_lse_merge_batch(dcp_ctx* ctx, int32_t dtype_bytes, int32_t n_groups,
                                int32_t head_dim, const int64_t* group_off, const void* outs,
                                const void* lses, void* merged, void* merged_lse, void* stream);

/* ---- K4 / K5: MoE dispatch / combine over peer pools ------------------------
 *
 * No reference symbol exists (the reference's MoE surface is the M list,
 * BindingConfig::moe_bound routing.hpp:18-19): parity is against our own CPU
 * restatement (oracle dcpora_moe_layer_f64), out_t = sum over its top-k
 * experts in ascending id of w * FFN_e(x_t).  Token t of an instance is the
 * t-th request of its M list.  Experts are partitioned contiguously:
 * rank = expert / (num_experts / world).  The expert FFN between receive and
 * combine_put is the caller's (a library GEMM; out of scope of this path). */
typedef struct dcp_moe dcp_moe;
typedef struct dcp_moe_config {
    int32_t world;
    int32_t self;
    int32_t hidden;       /* multiple of 8 */
    int32_t topk;         /* <= 16 */
    int32_t num_experts;  /* multiple of world */
    int32_t m_max;        /* max tokens per instance (<= 1024) */
    int32_t timeout_ms;   /* flag-wait bound; 0 = 10000 */
} dcp_moe_config;

/* Pools are double-buffered by step parity and fenced like dcp_xchg (every instance
 * calls dcp_moe_begin_step once per step; no instance runs more than one step ahead);
 * waits are bounded, a timeout is reported by dcp_moe_status as DCP_E_TIMEOUT. */
DCP_API int dcp_moe_create(dcp_ctx* ctx, const dcp_moe_config* cfg, dcp_moe** out);
DCP_API int dcp_moe_destroy(dcp_moe* x);
DCP_API int dcp_moe_ipc_handle(dcp_moe* x, void* handle64);
DCP_API int dcp_moe_open_peer_ipc(dcp_moe* x, int32_t peer, const void* handle64);
DCP_API int dcp_moe_set_peer_local(dcp_moe* x, int32_t peer, const dcp_moe* other);
DCP_API int dcp_moe_commit(dcp_moe* x);
DCP_API int dcp_moe_begin_step(dcp_moe* x, void* stream);
DCP_API int dcp_moe_status(dcp_moe* x, uint32_t* info);
/* int32 per received row of meta_rows: src token, n_local, (expert, weight bits) * topk */
DCP_API int32_t dcp_moe_meta_width(const dcp_moe* x);
/* K4: x_local bf16 [M][hidden] in M-row order, topk_idx int32 [M][topk], topk_w fp32
 * [M][topk] (device); *m_count_dev = M, e.g. dcp_instance_view.m_count_all + self (K7's
 * device M count, so the step needs no host round trip). */
DCP_API int dcp_moe_dispatch(dcp_moe* x, const void* x_local, const int32_t* topk_idx,
                             const float* topk_w, const int32_t* m_count_dev, void* stream);
/* dcp_moe_begin_step + dcp_moe_dispatch in ONE launch: K4 runs the step fence before its
 * first peer store and its last CTA advances the epoch.  Same results, one launch less. */
DCP_API int dcp_moe_step_dispatch(dcp_moe* x, const void* x_local, const int32_t* topk_idx,
                                  const float* topk_w, const int32_t* m_count_dev, void* stream);
/* dcp_moe_step_dispatch + dcp_moe_receive_regions in ONE launch: K4's last CTA waits for every
 * source's rows and writes the receive counts.  Only when the peers run concurrently (one
 * instance per process / GPU); instances sharing a GPU in one process use the two calls. */
DCP_API int dcp_moe_step_dispatch_recv(dcp_moe* x, const void* x_local, const int32_t* topk_idx,
                                       const float* topk_w, const int32_t* m_count_dev, void* stream);
/* K5a, region mode (the fast path): wait for every source; the received rows stay in
 * this instance's pool, source s's rows at x_region[s * m_max + j], j < count[s]
 * (meta likewise), for the expert stage to read in place.  Per-source counts and
 * offsets stay on the device (dcp_moe_recv_counts_dev).  Graph-capturable. */
DCP_API int dcp_moe_receive_regions(dcp_moe* x, void* stream);
/* Parity of the current step (host mirror of the epoch) and the region pointers of a
 * parity: bf16 [world][m_max][hidden], int32 [world][m_max][meta_width]. */
DCP_API int32_t dcp_moe_parity(const dcp_moe* x);
DCP_API int dcp_moe_regions(dcp_moe* x, int32_t parity, void** x_region, int32_t** meta_region);
/* K5a, compact mode: wait, then copy the received rows into x_rows (bf16
 * [world*m_max][hidden]) and meta_rows in (source, slot) order; returns the row count
 * and copies the per-source counts to host `counts`. */
DCP_API int32_t dcp_moe_receive(dcp_moe* x, void* x_rows, int32_t* meta_rows, int32_t* counts,
                                void* stream);
/* compact mode without the host read-back (stream-ordered, graph-capturable) */
DCP_API int dcp_moe_receive_async(dcp_moe* x, void* x_rows, int32_t* meta_rows, void* stream);
DCP_API const int32_t* dcp_moe_recv_counts_dev(const dcp_moe* x);
/* K5b: y rows back to each token's home; y_rows bf16 [R][hidden] in compact order, or
 * y_region bf16 [world][m_max][hidden] in region order. */
DCP_API int dcp_moe_combine_put(dcp_moe* x, const void* y_rows, void* stream);
DCP_API int dcp_moe_combine_put_regions(dcp_moe* x, const void* y_region, void* stream);
/* Gate-weighted identity expert stage (region mode): y_region[s][j] = (sum of row j's local
 * gate weights) * x_region[s][j] for every received row, reading this step's regions through
 * the device epoch (graph-safe).  The stand-in for the expert FFN in benches and graphs. */
DCP_API int dcp_moe_expert_identity(dcp_moe* x, void* y_region, void* stream);
/* K5c: out fp32 [M][hidden] = sum over ranks (ascending) of the returned partials. */
DCP_API int dcp_moe_combine_reduce(dcp_moe* x, float* out, void* stream);
/* K5b + K5c in one launch (region mode): the puts, then this instance's reduction once every
 * rank's rows have landed.  Bit-identical to dcp_moe_combine_put_regions + dcp_moe_combine_reduce.
 * Only when the peers run concurrently (one instance per process / GPU): instances sharing a
 * GPU in one process must use the two launches (the reduction spins on peers' puts). */
DCP_API int dcp_moe_combine_fused(dcp_moe* x, const void* y_region, float* out, void* stream);

/* ---- AOT step graphs (Alg. 2; ShapeSpace routing.hpp:60-85) --
 * One CUDA graph per M-bucket of ShapeSpace::default_space(), each replaying
 * this instance's routed step (epoch bump, K2, K1-routed, K3) over the same
 * pools (one shared pool for all graphs, as graph_memory_footprint models).
 * K2/K3 grids are the bucket's M^; K1 is persistent and reads N from device
 * memory, so buckets that differ only in N^ share one executable graph.
 * dcp_step_graph_launch picks bucket_shape(m_rows, n_rows) and replays it;
 * ShapeOverflow(-5) above (256, 512).  The view's device pointers must stay
 * valid (they are fixed offsets into the planner's routing buffers). */
typedef struct dcp_step_graph dcp_step_graph;
DCP_API int dcp_step_graph_create(dcp_ctx* ctx, dcp_xchg* x, const dcp_instance_view* v,
                                  const dcp_attn_args* a, dcp_step_graph** out);
DCP_API int dcp_step_graph_launch(dcp_step_graph* g, int32_t m_rows, int32_t n_rows, void* stream);
/* executable graphs captured / buckets in the shape space */
DCP_API int dcp_step_graph_count(const dcp_step_graph* g, int32_t* buckets);
DCP_API int dcp_step_graph_destroy(dcp_step_graph* g);

/* ---- Whole-layer AOT decode graphs (Alg. 2, 805-840, widened to the layer) ----
 * One instance's decode layer captured per (M-bucket, MoE step parity):
 *   [K7 dcp_planner_build_routing] -> dcp_xchg_begin_step -> K2 -> K1-routed -> K3
 *   -> dcp_moe_begin_step -> K4 dispatch -> K5a receive (regions) -> expert stage
 *   -> K5b combine_put (regions) -> K5c combine_reduce
 * and replayed once per decode step with dcp_layer_graph_launch.  All per-step metadata
 * is read on the device (K7 output), so a replay copies nothing in.  The M-bucket only
 * sizes the K2 / K3 grids (ShapeSpace M-hat ladder 8..m_max); any bucket is correct.
 * planner: optional; when set, K7 runs inside the graph (re-captured automatically if
 *   the planner's page arena was compacted since).
 * moe: optional (attention only when NULL); moe_x bf16 [m_max][hidden] (M-row order),
 *   topk_idx / topk_w [m_max][topk], y_region bf16 [world][m_max][hidden], moe_out fp32
 *   [m_max][hidden] — device buffers the graph reads / writes every replay.
 * expert: the expert stage, called at capture time to enqueue its work on `stream`
 *   (library GEMMs), with the receive regions of `parity` (bf16 [world][m_max][hidden],
 *   meta int32 [world][m_max][dcp_moe_meta_width]) and the device per-source counts; it
 *   must fill y_region.  NULL = dcp_moe_expert_identity.
 * Every instance of the step must replay its own graph (or run the same calls eagerly) once
 * per step; peers synchronise through the exchange flags as in the eager path. */
typedef void (*dcp_expert_fn)(void* user, void* stream, int32_t parity, void* x_region,
                              int32_t* meta_region, const int32_t* recv_counts_dev, void* y_region);
typedef struct dcp_layer_graph_desc {
    dcp_planner* planner;
    dcp_xchg* xchg;
    const dcp_instance_view* view;
    const dcp_attn_args* attn;       /* bf16 routed K1 arguments (kv_pool, workspace, scale) */
    dcp_moe* moe;
    const void* moe_x;
    const int32_t* topk_idx;
    const float* topk_w;
    void* y_region;
    float* moe_out;
    dcp_expert_fn expert;
    void* expert_user;
    int32_t fused_step;              /* 1: the attention sub-step is one dcp_decode_step_fused launch */
} dcp_layer_graph_desc;
typedef struct dcp_layer_graph dcp_layer_graph;
DCP_API int dcp_layer_graph_create(dcp_ctx* ctx, const dcp_layer_graph_desc* desc, dcp_layer_graph** out);
/* m_rows: this step's M (or any upper bound <= m_max) picks the bucket. */
DCP_API int dcp_layer_graph_launch(dcp_layer_graph* g, int32_t m_rows, void* stream);
/* Returns the executable graph count; buckets / captures (1 + re-captures) if non-NULL. */
DCP_API int dcp_layer_graph_info(const dcp_layer_graph* g, int32_t* buckets, int32_t* captures);
DCP_API int dcp_layer_graph_destroy(dcp_layer_graph* g);

/* ---- K8: kv_append — the decode step's new K/V into the paged pools ----------
 * After dcp_planner_append_token + dcp_planner_build_routing, write each
 * request's new-token K and V (bf16 [M][2][num_kv_heads][head_dim], in the
 * M-row order of `instance`, i.e. produced at the MoE binding) into the frame
 * and slot that append_token chose (page_table.cpp:86-121) — on whichever
 * instance holds it.  pools[s] (host array of W device pointers) is instance
 * s's KV pool [frames][2][num_kv_heads][page_size][head_dim] as addressable
 * from this device (local pointer, or a peer / CUDA-IPC mapping). */
DCP_API int dcp_kv_append(dcp_planner* pl, int32_t instance, const void* kv_new, void* const* pools,
                          int32_t num_kv_heads, int32_t head_dim, void* stream);

/* ---- KV migration: prefill -> decode (steps MIGRATE / TRANSFER) ----
 * After dcp_planner_step admitted requests ids[0..n) (GlobalPageTable::allocate,
 * page_table.cpp:9-49, chose their frames), copy each request's prefill K and V
 * — src_k[i], src_v[i]: [seq_len][num_kv_heads][head_dim] elements of elem_bytes
 * (2 = bf16, 4 = fp32), readable from this device (local or peer / CUDA-IPC
 * mapped) — into those frames: logical page j, held by (instance, frame) of the
 * page table, receives the request's tokens [sum of the earlier pages' fills, +
 * fill_j), i.e. each kv_binding member its split in order.  pools[s] (host array
 * of W device pointers) is instance s's pool [frames][2][num_kv_heads][page][head_dim]
 * as addressable from this device; stores to remote instances go over NVLink.
 * One kernel launch, stream-ordered.  UnknownRequest(-2) for an id the planner
 * does not track, InvalidArgument for one that holds no pages. */
DCP_API int dcp_kv_migrate(dcp_planner* pl, const int64_t* ids, int32_t n, const void* const* src_k,
                           const void* const* src_v, void* const* pools, int32_t num_kv_heads,
                           int32_t head_dim, int32_t elem_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DCP_CAPI_H_ */
