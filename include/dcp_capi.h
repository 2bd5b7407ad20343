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
    DCP_E_CUDA = -10                 /* CUDA runtime / driver failure  */
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
 * Compiled shapes: head_dim 128, page_size 16, (num_kv_heads, group) in
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

/* Number of kernel launches the last dcp_splitkv_decode_attn issued (for the
 * bench's gpu_launches accounting). */
DCP_API int dcp_attn_launches_per_call(void);

#ifdef __cplusplus
}
#endif
#endif /* DCP_CAPI_H_ */
