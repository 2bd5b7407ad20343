// SPDX-License-Identifier: Apache-2.0
// C ABI: context + K1/K9 split-KV paged decode attention (dcp_capi.h).
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "capi_common.cuh"
#include "splitkv_decode.cuh"
#include "splitkv_decode_f32.cuh"
#include "xchg_internal.cuh"

namespace dcp {

static thread_local std::string g_err;

void set_error(const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// 2-D view of the paged pool: rows = frame*2*HKV*16 + (kv*HKV + head)*16 + tok,
// columns = head_dim (bf16).  Box = 64 columns (128 B, 128B swizzle) x all
// rows of one frame.
static int kv_tensor_map(dcp_ctx* ctx, const void* pool, int64_t frames, int hkv, int d,
                         const CUtensorMap** out, bool split, int page = 16) {
    for (auto& e : ctx->kv_maps) {
        if (e.base == pool && e.frames == frames && e.hkv == hkv && e.d == d && e.split == split &&
            e.page == page) {
            *out = &e.map;
            return DCP_OK;
        }
    }
    auto fn = encode_fn();
    DCP_REQUIRE(fn != nullptr, DCP_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    auto& e = ctx->kv_maps[ctx->kv_map_next];
    ctx->kv_map_next = (ctx->kv_map_next + 1) % 4;
    CUresult r;
    if (!split) {
        // whole-frame ring: rows = frame*2*HKV*16 + (kv*HKV + head)*16 + tok, box = one frame
        const int rows_per_frame = 2 * hkv * 16;
        cuuint64_t dims[2] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(frames) * rows_per_frame};
        cuuint64_t strides[1] = {static_cast<cuuint64_t>(d) * 2};
        cuuint32_t box[2] = {64, static_cast<cuuint32_t>(rows_per_frame)};
        cuuint32_t estr[2] = {1, 1};
        r = fn(&e.map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(pool), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    } else {
        // split ring: (d, token-in-page, frame*2*HKV + kv*HKV + head); box = 16 tokens of every head
        cuuint64_t dims[3] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(page),
                              static_cast<cuuint64_t>(frames) * 2 * hkv};
        cuuint64_t strides[2] = {static_cast<cuuint64_t>(d) * 2, static_cast<cuuint64_t>(page) * d * 2};
        cuuint32_t box[3] = {64, 16, static_cast<cuuint32_t>(hkv)};
        cuuint32_t estr[3] = {1, 1, 1};
        r = fn(&e.map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(pool), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    }
    if (r != CUDA_SUCCESS) {
        e.base = nullptr;
        set_error("cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
        return DCP_E_CUDA;
    }
    e.base = pool;
    e.frames = frames;
    e.hkv = hkv;
    e.d = d;
    e.split = split;
    e.page = page;
    *out = &e.map;
    return DCP_OK;
}

template <int HKV, int G, bool SPLIT, int PAGE = 16>
static int ensure_attr(dcp_ctx* ctx) {
    using C = DecodeCfg<HKV, G, SPLIT, PAGE>;
    static uint64_t attr_done = 0;  // per-instantiation bit per device
    if (!(attr_done >> (ctx->device & 63) & 1)) {
        DCP_CUDA_TRY(cudaFuncSetAttribute(splitkv_decode_kernel<HKV, G, SPLIT, PAGE>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
        attr_done |= uint64_t(1) << (ctx->device & 63);
    }
    return DCP_OK;
}

template <int HKV, int G, bool SPLIT, int PAGE = 16>
static int launch_decode(dcp_ctx* ctx, const CUtensorMap* map, const AttnParams& prm,
                         cudaStream_t stream) {
    using C = DecodeCfg<HKV, G, SPLIT, PAGE>;
    if (int rc = ensure_attr<HKV, G, SPLIT, PAGE>(ctx)) return rc;
    splitkv_decode_kernel<HKV, G, SPLIT, PAGE><<<ctx->num_sms, C::THREADS, C::SMEM, stream>>>(*map, prm);
    DCP_CUDA_TRY(cudaGetLastError());
    return DCP_OK;
}

// K1 ring variant: env DCP_K1_SPLIT=1 selects split half-frame stages (default: whole frames).
static bool k1_split() {
    static int v = -1;
    if (v < 0) {
        const char* e = std::getenv("DCP_K1_SPLIT");
        v = e ? (std::atoi(e) != 0) : 0;
    }
    return v != 0;
}

static long long* g_k1_trace = nullptr;

static int dispatch_decode(dcp_ctx* ctx, const CUtensorMap* map, const AttnParams& prm0, int hkv, int G,
                           cudaStream_t s, int page = 16) {
    const bool sp = k1_split();
    AttnParams prm = prm0;
    prm.trace = g_k1_trace;
#define DCP_K1(H_, G_)                                                                                  \
    if (hkv == H_ && G == G_) {                                                                          \
        if (page == 32) return launch_decode<H_, G_, true, 32>(ctx, map, prm, s);                        \
        if (page == 64) return launch_decode<H_, G_, true, 64>(ctx, map, prm, s);                        \
        return sp ? launch_decode<H_, G_, true>(ctx, map, prm, s) : launch_decode<H_, G_, false>(ctx, map, prm, s); \
    }
    DCP_K1(8, 4)
    DCP_K1(4, 8)
    DCP_K1(8, 1)
    DCP_K1(2, 16)
    DCP_K1(1, 16)
#undef DCP_K1
    set_error("unsupported (num_kv_heads=%d, group=%d)", hkv, G);
    return DCP_E_UNSUPPORTED;
}

}  // namespace dcp

using namespace dcp;

int dcp_attn_prepare(dcp_ctx* ctx, int hkv, int G, int page) {
    const bool sp = k1_split();
#define DCP_K1A(H_, G_)                                                               \
    if (hkv == H_ && G == G_) {                                                       \
        if (page == 32) return ensure_attr<H_, G_, true, 32>(ctx);                    \
        if (page == 64) return ensure_attr<H_, G_, true, 64>(ctx);                    \
        return sp ? ensure_attr<H_, G_, true>(ctx) : ensure_attr<H_, G_, false>(ctx); \
    }
    DCP_K1A(8, 4)
    DCP_K1A(4, 8)
    DCP_K1A(8, 1)
    DCP_K1A(2, 16)
    DCP_K1A(1, 16)
#undef DCP_K1A
    set_error("unsupported (num_kv_heads=%d, group=%d)", hkv, G);
    return DCP_E_UNSUPPORTED;
}

extern "C" {

const char* dcp_last_error(void) { return g_err.c_str(); }
const char* dcp_version(void) { return "dcp-b200 0.1 (sm_100a)"; }

int dcp_ctx_create(int device, dcp_ctx** out) {
    DCP_REQUIRE(out != nullptr, DCP_E_INVALID_ARG, "out is NULL");
    int n = 0;
    DCP_CUDA_TRY(cudaGetDeviceCount(&n));
    DCP_REQUIRE(device >= 0 && device < n, DCP_E_INVALID_ARG, "device %d of %d", device, n);
    DCP_CUDA_TRY(cudaSetDevice(device));
    auto* c = new dcp_ctx();
    c->device = device;
    cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
    cudaDeviceGetAttribute(&c->cc_major, cudaDevAttrComputeCapabilityMajor, device);
    cudaDeviceGetAttribute(&c->cc_minor, cudaDevAttrComputeCapabilityMinor, device);
    if (c->cc_major != 10) {
        set_error("device %d is sm_%d%d; this library is built for sm_100a only", device,
                  c->cc_major, c->cc_minor);
        delete c;
        return DCP_E_UNSUPPORTED;
    }
    *out = c;
    return DCP_OK;
}

int dcp_ctx_destroy(dcp_ctx* ctx) {
    delete ctx;
    return DCP_OK;
}

int dcp_ctx_num_sms(const dcp_ctx* ctx) { return ctx ? ctx->num_sms : 0; }

static __global__ void device_sleep_kernel(int64_t ns) {
    int64_t g0, now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
    do {
        __nanosleep(2000);
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    } while (now - g0 < ns);
}

int dcp_device_sleep(dcp_ctx* ctx, int32_t us, void* stream) {
    DCP_REQUIRE(ctx && us >= 0 && us <= 1000000, DCP_E_INVALID_ARG, "sleep %d us", us);
    device_sleep_kernel<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>((int64_t)us * 1000);
    DCP_CUDA_TRY(cudaGetLastError());
    return DCP_OK;
}

int dcp_copy_to_host(void* dst, const void* src, size_t bytes) {
    DCP_REQUIRE(dst && (src || bytes == 0), DCP_E_INVALID_ARG, "NULL pointer");
    if (bytes) DCP_CUDA_TRY(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
    return DCP_OK;
}

size_t dcp_attn_workspace_bytes(const dcp_ctx* ctx, int32_t num_shards, int32_t num_q_heads,
                                int32_t head_dim) {
    if (!ctx || num_shards < 0 || num_q_heads <= 0 || head_dim <= 0) return 0;
    const size_t slots = 2 * static_cast<size_t>(ctx->num_sms);
    size_t b = slots * num_q_heads * head_dim * sizeof(float);  // ws_acc
    b += slots * num_q_heads * 2 * sizeof(float);               // ws_ml
    b += static_cast<size_t>(num_shards) * sizeof(int32_t);     // counters
    return (b + 255) & ~size_t(255);
}

int dcp_attn_launches_per_call(void) { return 1; }

/* Debug: per-CTA globaltimer stamps of the next K1 launches into a device buffer of
 * num_sms x 8 int64 (NULL = off): entry, first ring stage, segment end, ticket, merge end,
 * exit, SM id, pages. */
int dcp_k1_set_trace(void* dev_buf) {
    g_k1_trace = static_cast<long long*>(dev_buf);
    return DCP_OK;
}

int dcp_splitkv_decode_attn(dcp_ctx* ctx, const dcp_attn_args* a, void* stream) {
    DCP_NVTX("K1 splitkv_decode");
    DCP_REQUIRE(ctx && a, DCP_E_INVALID_ARG, "NULL ctx/args");
    DCP_REQUIRE(a->num_shards >= 0, DCP_E_INVALID_ARG, "num_shards < 0");
    if (a->num_shards == 0) return DCP_OK;
    DCP_REQUIRE(a->head_dim == 128, DCP_E_UNSUPPORTED, "head_dim %d (compiled: 128)", a->head_dim);
    DCP_REQUIRE(a->page_size == 16 || a->page_size == 32 || a->page_size == 64, DCP_E_UNSUPPORTED,
                "page_size %d (compiled: 16, 32, 64)", a->page_size);
    DCP_REQUIRE(a->num_kv_heads > 0 && a->num_q_heads % a->num_kv_heads == 0, DCP_E_INVALID_ARG,
                "num_q_heads %d not a multiple of num_kv_heads %d", a->num_q_heads, a->num_kv_heads);
    DCP_REQUIRE(a->q && a->kv_pool && a->block_table && a->cu_pages && a->shard_len && a->out &&
                    a->lse && a->workspace,
                DCP_E_INVALID_ARG, "NULL device pointer in dcp_attn_args");
    DCP_REQUIRE((reinterpret_cast<uintptr_t>(a->kv_pool) & 15) == 0, DCP_E_INVALID_ARG,
                "kv_pool must be 16-byte aligned");
    DCP_REQUIRE(a->num_frames > 0, DCP_E_INVALID_ARG, "num_frames <= 0");
    const size_t need = dcp_attn_workspace_bytes(ctx, a->num_shards, a->num_q_heads, a->head_dim);
    DCP_REQUIRE(a->workspace_bytes >= need, DCP_E_INVALID_ARG, "workspace %zu < %zu bytes",
                a->workspace_bytes, need);
    const int G = a->num_q_heads / a->num_kv_heads;

    const CUtensorMap* map = nullptr;
    const bool split = k1_split() || a->page_size != 16;
    int rc = kv_tensor_map(ctx, a->kv_pool, a->num_frames, a->num_kv_heads, a->head_dim, &map, split, a->page_size);
    if (rc) return rc;

    AttnParams prm{};
    prm.q = static_cast<const __nv_bfloat16*>(a->q);
    prm.block_table = a->block_table;
    prm.cu_pages = a->cu_pages;
    prm.shard_len = a->shard_len;
    prm.page_fill = a->page_fill;
    prm.out = a->out;
    prm.lse = a->lse;
    const size_t slots = 2 * static_cast<size_t>(ctx->num_sms);
    char* ws = static_cast<char*>(a->workspace);
    prm.ws_acc = reinterpret_cast<float*>(ws);
    ws += slots * a->num_q_heads * a->head_dim * sizeof(float);
    prm.ws_ml = reinterpret_cast<float*>(ws);
    ws += slots * a->num_q_heads * 2 * sizeof(float);
    prm.counters = reinterpret_cast<int32_t*>(ws);
    prm.num_shards = a->num_shards;
    prm.scale_log2 = a->scale * 1.4426950408889634f;

    return dispatch_decode(ctx, map, prm, a->num_kv_heads, G, static_cast<cudaStream_t>(stream), a->page_size);
}

static int decode_routed(dcp_ctx* ctx, dcp_xchg* x, const dcp_instance_view* v, const dcp_attn_args* a,
                         uint32_t fuse, void* stream) {
    DCP_REQUIRE(ctx && x && v && a, DCP_E_INVALID_ARG, "NULL argument");
    DCP_REQUIRE(v->instance == x->cfg.self, DCP_E_INVALID_ARG, "view/instance mismatch");
    DCP_REQUIRE(v->n_rows <= x->cfg.n_max, DCP_E_SHAPE_OVERFLOW, "N %d > n_max %d", v->n_rows, x->cfg.n_max);
    DCP_REQUIRE(a->head_dim == 128 && (a->page_size == 16 || a->page_size == 32 || a->page_size == 64),
                DCP_E_UNSUPPORTED, "head_dim/page_size");
    DCP_REQUIRE(a->num_q_heads == x->cfg.num_q_heads && a->head_dim == x->cfg.q_dim &&
                    a->head_dim == x->cfg.o_dim && x->cfg.q_elem_bytes == 2,
                DCP_E_INVALID_ARG, "exchange pool shape differs from the bf16 attention shape");
    DCP_REQUIRE(a->kv_pool && a->workspace && a->num_frames > 0, DCP_E_INVALID_ARG, "kv_pool/workspace");
    DCP_REQUIRE(a->num_kv_heads > 0 && a->num_q_heads % a->num_kv_heads == 0, DCP_E_INVALID_ARG, "heads");
    const size_t need = dcp_attn_workspace_bytes(ctx, x->cfg.n_max, a->num_q_heads, a->head_dim);
    DCP_REQUIRE(a->workspace_bytes >= need, DCP_E_INVALID_ARG, "workspace %zu < %zu", a->workspace_bytes, need);
    const CUtensorMap* map = nullptr;
    const bool split = k1_split() || a->page_size != 16;
    int rc = kv_tensor_map(ctx, a->kv_pool, a->num_frames, a->num_kv_heads, a->head_dim, &map, split, a->page_size);
    if (rc) return rc;
    AttnParams prm{};
    prm.q = nullptr;  // from the receive pool, by epoch parity
    prm.block_table = v->block_table;
    prm.cu_pages = v->cu_pages;
    prm.shard_len = v->shard_len;
    prm.page_fill = v->page_fill;
    prm.out = nullptr;
    prm.lse = nullptr;
    char* ws = static_cast<char*>(a->workspace);
    const size_t slots = 2 * static_cast<size_t>(ctx->num_sms);
    prm.ws_acc = reinterpret_cast<float*>(ws);
    ws += slots * a->num_q_heads * a->head_dim * sizeof(float);
    prm.ws_ml = reinterpret_cast<float*>(ws);
    ws += slots * a->num_q_heads * 2 * sizeof(float);
    prm.counters = reinterpret_cast<int32_t*>(ws);
    prm.num_shards = 0;
    prm.scale_log2 = a->scale * 1.4426950408889634f;
    prm.xp = x->dev;
    prm.n_mrow = v->n_mrow;
    prm.n_moe = v->n_moe;
    prm.num_shards_ptr = v->n_count_dev;
    prm.total_pages_ptr = v->total_pages_dev;
    prm.fuse = fuse;
    if (fuse) {
        prm.q_local = x->q_local;
        prm.m_count = v->m_count_all;
        prm.m_nrow = v->m_nrow;
        prm.m_k = v->m_k;
        prm.m_kv = v->m_kv;
        prm.mout = x->out;
        prm.mout_lse = x->out_lse;
        prm.exit_ticket = x->exit_ticket;
    }
    return dispatch_decode(ctx, map, prm, a->num_kv_heads, a->num_q_heads / a->num_kv_heads,
                           static_cast<cudaStream_t>(stream), a->page_size);
}

int dcp_decode_attn_routed(dcp_ctx* ctx, dcp_xchg* x, const dcp_instance_view* v, const dcp_attn_args* a,
                           void* stream) {
    DCP_NVTX("K1 routed");
    return decode_routed(ctx, x, v, a, 0u, stream);
}

int dcp_decode_step_fused(dcp_ctx* ctx, dcp_xchg* x, const dcp_instance_view* v, const dcp_attn_args* a,
                          void* stream) {
    DCP_NVTX("DCP fused step (fence + K2 + K1 + K3)");
    DCP_REQUIRE(x && x->committed, DCP_E_INVALID_ARG, "NULL or uncommitted exchange (dcp_xchg_commit)");
    DCP_REQUIRE(v && v->m_rows <= x->cfg.m_max, DCP_E_SHAPE_OVERFLOW, "M %d > m_max %d", v ? v->m_rows : 0,
                x->cfg.m_max);
    return decode_routed(ctx, x, v, a, FUSE_STEP | FUSE_ROUTE | FUSE_MERGE, stream);
}

// ---- K1-f32 ------------------------------------------------------------------------------

static int launch_f32(dcp_ctx* ctx, const AttnF32Params& prm, int G, cudaStream_t s) {
    const dim3 block(prm.hkv * 32);
    switch (G) {
        case 1: splitkv_decode_f32_kernel<1><<<ctx->num_sms, block, 0, s>>>(prm); break;
        case 2: splitkv_decode_f32_kernel<2><<<ctx->num_sms, block, 0, s>>>(prm); break;
        case 4: splitkv_decode_f32_kernel<4><<<ctx->num_sms, block, 0, s>>>(prm); break;
        case 8: splitkv_decode_f32_kernel<8><<<ctx->num_sms, block, 0, s>>>(prm); break;
        default: set_error("fp32 path: group %d (compiled 1, 2, 4, 8)", G); return DCP_E_UNSUPPORTED;
    }
    DCP_CUDA_TRY(cudaGetLastError());
    return DCP_OK;
}

static int f32_common(dcp_ctx* ctx, const dcp_attn_args* a, AttnF32Params& prm) {
    DCP_REQUIRE(a->head_dim == 128, DCP_E_UNSUPPORTED, "head_dim %d (compiled: 128)", a->head_dim);
    DCP_REQUIRE(a->num_kv_heads >= 1 && a->num_kv_heads <= 8 && a->num_q_heads % a->num_kv_heads == 0,
                DCP_E_UNSUPPORTED, "fp32 path: num_kv_heads %d (1..8), num_q_heads %d", a->num_kv_heads,
                a->num_q_heads);
    DCP_REQUIRE(a->page_size >= 1 && a->page_size <= 255, DCP_E_UNSUPPORTED, "page_size %d", a->page_size);
    DCP_REQUIRE(a->kv_pool && a->workspace && a->num_frames > 0, DCP_E_INVALID_ARG, "kv_pool/workspace");
    DCP_REQUIRE((reinterpret_cast<uintptr_t>(a->kv_pool) & 15) == 0, DCP_E_INVALID_ARG,
                "kv_pool must be 16-byte aligned");
    prm.kv = static_cast<const float*>(a->kv_pool);
    char* ws = static_cast<char*>(a->workspace);
    const size_t slots = 2 * static_cast<size_t>(ctx->num_sms);
    prm.ws_acc = reinterpret_cast<float*>(ws);
    ws += slots * a->num_q_heads * a->head_dim * sizeof(float);
    prm.ws_ml = reinterpret_cast<float*>(ws);
    ws += slots * a->num_q_heads * 2 * sizeof(float);
    prm.counters = reinterpret_cast<int32_t*>(ws);
    prm.hkv = a->num_kv_heads;
    prm.page = a->page_size;
    prm.scale = a->scale;
    return DCP_OK;
}

int dcp_splitkv_decode_attn_f32(dcp_ctx* ctx, const dcp_attn_args* a, void* stream) {
    DCP_NVTX("K1 splitkv_decode f32");
    DCP_REQUIRE(ctx && a, DCP_E_INVALID_ARG, "NULL ctx/args");
    DCP_REQUIRE(a->num_shards >= 0, DCP_E_INVALID_ARG, "num_shards < 0");
    if (a->num_shards == 0) return DCP_OK;
    DCP_REQUIRE(a->q && a->block_table && a->cu_pages && a->shard_len && a->out && a->lse, DCP_E_INVALID_ARG,
                "NULL device pointer in dcp_attn_args");
    const size_t need = dcp_attn_workspace_bytes(ctx, a->num_shards, a->num_q_heads, a->head_dim);
    DCP_REQUIRE(a->workspace_bytes >= need, DCP_E_INVALID_ARG, "workspace %zu < %zu bytes", a->workspace_bytes,
                need);
    AttnF32Params prm{};
    if (int rc = f32_common(ctx, a, prm)) return rc;
    prm.q = static_cast<const float*>(a->q);
    prm.block_table = a->block_table;
    prm.cu_pages = a->cu_pages;
    prm.shard_len = a->shard_len;
    prm.page_fill = a->page_fill;
    prm.out = a->out;
    prm.lse = a->lse;
    prm.num_shards = a->num_shards;
    return launch_f32(ctx, prm, a->num_q_heads / a->num_kv_heads, static_cast<cudaStream_t>(stream));
}

int dcp_decode_attn_routed_f32(dcp_ctx* ctx, dcp_xchg* x, const dcp_instance_view* v, const dcp_attn_args* a,
                               void* stream) {
    DCP_REQUIRE(ctx && x && v && a, DCP_E_INVALID_ARG, "NULL argument");
    DCP_REQUIRE(v->instance == x->cfg.self, DCP_E_INVALID_ARG, "view/instance mismatch");
    DCP_REQUIRE(v->n_rows <= x->cfg.n_max, DCP_E_SHAPE_OVERFLOW, "N %d > n_max %d", v->n_rows, x->cfg.n_max);
    DCP_REQUIRE(a->num_q_heads == x->cfg.num_q_heads && a->head_dim == x->cfg.q_dim && a->head_dim == x->cfg.o_dim &&
                    x->cfg.q_elem_bytes == 4,
                DCP_E_INVALID_ARG, "exchange pool shape differs from the fp32 attention shape");
    const size_t need = dcp_attn_workspace_bytes(ctx, x->cfg.n_max, a->num_q_heads, a->head_dim);
    DCP_REQUIRE(a->workspace_bytes >= need, DCP_E_INVALID_ARG, "workspace %zu < %zu", a->workspace_bytes, need);
    AttnF32Params prm{};
    if (int rc = f32_common(ctx, a, prm)) return rc;
    prm.block_table = v->block_table;
    prm.cu_pages = v->cu_pages;
    prm.shard_len = v->shard_len;
    prm.page_fill = v->page_fill;
    prm.xp = x->dev;
    prm.n_mrow = v->n_mrow;
    prm.n_moe = v->n_moe;
    prm.num_shards_ptr = v->n_count_dev;
    return launch_f32(ctx, prm, a->num_q_heads / a->num_kv_heads, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
