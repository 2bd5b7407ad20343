// SPDX-License-Identifier: Apache-2.0
// C ABI: K10 MLA split-KV paged decode attention (dcp_capi.h, dcp_mla_*).
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "capi_common.cuh"
#include "mla_decode.cuh"
#include "xchg_internal.cuh"

namespace dcp {

static long long* g_mla_trace = nullptr;

static PFN_cuTensorMapEncodeTiled_v12000 mla_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    });
    return fn;
}

// Pairs the persistent kernel runs: one cluster of 2 per TPC that can hold it.
template <int PAGE>
static int mla_pairs(dcp_ctx* ctx, int* out) {
    static int cached[64] = {0};
    int& c = cached[ctx->device & 63];
    if (c == 0) {
        DCP_CUDA_TRY(cudaFuncSetAttribute(mla::mla_decode_kernel<PAGE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          mla::SMEM));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(ctx->num_sms & ~1);
        cfg.blockDim = dim3(mla::THREADS);
        cfg.dynamicSmemBytes = mla::SMEM;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int n = 0;
        DCP_CUDA_TRY(cudaOccupancyMaxActiveClusters(&n, mla::mla_decode_kernel<PAGE>, &cfg));
        c = n > 0 ? (n < ctx->num_sms / 2 ? n : ctx->num_sms / 2) : ctx->num_sms / 2;
    }
    *out = c;
    return DCP_OK;
}

// Routed launch context (dcp_mla_decode_attn_routed); NULL for a local call.
struct MlaRoute {
    dcp_xchg* x;
    const dcp_instance_view* v;
};

template <int PAGE>
static int mla_launch(dcp_ctx* ctx, const dcp_mla_args* a, cudaStream_t stream, const MlaRoute* rt = nullptr) {
    auto fn = mla_encode_fn();
    DCP_REQUIRE(fn != nullptr, DCP_E_CUDA, "cuTensorMapEncodeTiled unavailable");
    int pairs = 0;
    if (int rc = mla_pairs<PAGE>(ctx, &pairs)) return rc;

    CUtensorMap qmap, kvq, kvp;
    {
        // routed: both parities of the receive pool, rows (parity * n_max + r) * H + head
        const void* qbase = rt ? static_cast<const void*>(rt->x->pool + rt->x->host.off_qrecv) : a->q;
        const cuuint64_t qrows = rt ? 2ull * rt->x->cfg.n_max * mla::H : static_cast<cuuint64_t>(a->num_shards) * mla::H;
        cuuint64_t dims[2] = {mla::DK, qrows};
        cuuint64_t strides[1] = {mla::DK * 2};
        cuuint32_t box[2] = {64, 64};
        cuuint32_t estr[2] = {1, 1};
        CUresult r = fn(&qmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(qbase), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        DCP_REQUIRE(r == CUDA_SUCCESS, DCP_E_CUDA, "q tensor map (%d)", static_cast<int>(r));
    }
    // paged cache as (column, token-in-page, frame); QK boxes take min(PAGE, HT) rows, PV boxes min(PAGE, 32)
    for (int which = 0; which < 2; ++which) {
        const cuuint32_t rows = which == 0 ? (PAGE < mla::HT ? PAGE : mla::HT) : (PAGE < 32 ? PAGE : 32);
        cuuint64_t dims[3] = {mla::DK, PAGE, static_cast<cuuint64_t>(a->num_frames)};
        cuuint64_t strides[2] = {mla::DK * 2, static_cast<cuuint64_t>(PAGE) * mla::DK * 2};
        cuuint32_t box[3] = {64, rows, 1};
        cuuint32_t estr[3] = {1, 1, 1};
        CUresult r = fn(which == 0 ? &kvq : &kvp, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(a->kv_pool),
                        dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        DCP_REQUIRE(r == CUDA_SUCCESS, DCP_E_CUDA, "kv tensor map (%d)", static_cast<int>(r));
    }
    mla::MlaParams p{};
    p.block_table = a->block_table;
    p.cu_pages = a->cu_pages;
    p.shard_len = a->shard_len;
    p.page_fill = a->page_fill;
    p.out = a->out;
    p.lse = a->lse;
    const size_t slots = 2 * static_cast<size_t>(ctx->num_sms / 2);
    char* ws = static_cast<char*>(a->workspace);
    p.ws_acc = reinterpret_cast<float*>(ws);
    ws += slots * mla::H * mla::DL * sizeof(float);
    p.ws_ml = reinterpret_cast<float*>(ws);
    ws += slots * mla::H * 2 * sizeof(float);
    p.cu_tiles = reinterpret_cast<int32_t*>(ws);
    ws += (static_cast<size_t>(a->num_shards) + 1) * sizeof(int32_t);
    p.pair_t0 = reinterpret_cast<int32_t*>(ws);
    ws += (static_cast<size_t>(pairs) + 1) * sizeof(int32_t);
    p.num_pairs = pairs;
    if (rt) {
        p.xp = rt->x->dev;
        p.n_mrow = rt->v->n_mrow;
        p.n_moe = rt->v->n_moe;
        p.num_shards_ptr = rt->v->n_count_dev;
        p.q_rows = rt->x->cfg.n_max;
        p.tickets = reinterpret_cast<int32_t*>(ws);
        DCP_CUDA_TRY(cudaMemsetAsync(p.tickets, 0, static_cast<size_t>(a->num_shards) * sizeof(int32_t), stream));
    }
    static const int seg_tiles = [] { const char* e = std::getenv("DCP_MLA_SEG_TILES"); return e ? std::atoi(e) : 4; }();
    p.seg_tiles = seg_tiles;
    p.num_shards = a->num_shards;
    p.num_frames = static_cast<int32_t>(a->num_frames);
    p.scale_log2 = a->scale * 1.4426950408889634f;
#ifdef DCP_MLA_DBG
    p.dbg = DCP_MLA_DBG;  // bottleneck experiments only: a -DDCP_MLA_DBG=n build produces wrong results
#else
    p.dbg = 0;
#endif
    p.trace = g_mla_trace;

    mla::mla_tile_scan_kernel<PAGE><<<1, 1024, 0, stream>>>(p);
    DCP_CUDA_TRY(cudaGetLastError());
    // PDL chain: scan -> decode (prologue overlaps the scan) -> merge (launch overlaps the decode tail)
    DCP_CUDA_TRY(launch_pdl(mla::mla_decode_kernel<PAGE>, dim3(2 * pairs), dim3(mla::THREADS), mla::SMEM, stream,
                            qmap, kvq, kvp, p));
    DCP_CUDA_TRY(launch_pdl(mla::mla_merge_kernel, dim3(a->num_shards, mla::H / 16, mla::MERGE_QUARTERS), dim3(512), 0,
                            stream, p, pairs));
    return DCP_OK;
}

}  // namespace dcp

using namespace dcp;

extern "C" {

size_t dcp_mla_workspace_bytes(const dcp_ctx* ctx, int32_t num_shards) {
    if (!ctx || num_shards < 0) return 0;
    const size_t slots = 2 * static_cast<size_t>(ctx->num_sms / 2);
    size_t b = slots * mla::H * mla::DL * sizeof(float);          // ws_acc
    b += slots * mla::H * 2 * sizeof(float);                      // ws_ml
    b += (static_cast<size_t>(num_shards) + 1) * sizeof(int32_t); // cu_tiles
    b += (slots / 2 + 1) * sizeof(int32_t);                       // pair_t0
    b += static_cast<size_t>(num_shards) * sizeof(int32_t);       // routed-mode merge tickets
    return (b + 255) & ~size_t(255);
}

int dcp_mla_launches_per_call(void) { return 3; }

/* Debug: globaltimer stamps of pair 0 into a device buffer of 256 x 8 int64 (NULL = off). */
int dcp_mla_set_trace(void* dev_buf) {
    g_mla_trace = static_cast<long long*>(dev_buf);
    return DCP_OK;
}

int dcp_mla_decode_attn(dcp_ctx* ctx, const dcp_mla_args* a, void* stream) {
    DCP_NVTX("K10 mla_decode");
    DCP_REQUIRE(ctx && a, DCP_E_INVALID_ARG, "NULL ctx/args");
    DCP_REQUIRE(a->num_shards >= 0, DCP_E_INVALID_ARG, "num_shards < 0");
    if (a->num_shards == 0) return DCP_OK;
    DCP_REQUIRE(a->num_q_heads == mla::H && a->kv_lora_rank == mla::DL && a->rope_dim == mla::DR, DCP_E_UNSUPPORTED,
                "MLA shape (heads %d, kv_lora_rank %d, rope_dim %d); compiled: 128 / 512 / 64", a->num_q_heads,
                a->kv_lora_rank, a->rope_dim);
    DCP_REQUIRE(a->page_size == 16 || a->page_size == 32 || a->page_size == 64, DCP_E_UNSUPPORTED,
                "page_size %d (compiled: 16, 32, 64)", a->page_size);
    DCP_REQUIRE(a->q && a->kv_pool && a->block_table && a->cu_pages && a->shard_len && a->out && a->lse &&
                    a->workspace,
                DCP_E_INVALID_ARG, "NULL device pointer in dcp_mla_args");
    DCP_REQUIRE((reinterpret_cast<uintptr_t>(a->kv_pool) & 15) == 0 && (reinterpret_cast<uintptr_t>(a->q) & 15) == 0,
                DCP_E_INVALID_ARG, "q and kv_pool must be 16-byte aligned");
    DCP_REQUIRE(a->num_frames > 0 && a->num_frames < (int64_t(1) << 31), DCP_E_INVALID_ARG, "num_frames");
    DCP_REQUIRE(static_cast<int64_t>(a->num_shards) * mla::H < (int64_t(1) << 31), DCP_E_INVALID_ARG,
                "num_shards too large");
    const size_t need = dcp_mla_workspace_bytes(ctx, a->num_shards);
    DCP_REQUIRE(a->workspace_bytes >= need, DCP_E_INVALID_ARG, "workspace %zu < %zu bytes", a->workspace_bytes,
                need);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (a->page_size == 16) return mla_launch<16>(ctx, a, s);
    if (a->page_size == 32) return mla_launch<32>(ctx, a, s);
    return mla_launch<64>(ctx, a, s);
}

int dcp_mla_decode_attn_routed(dcp_ctx* ctx, dcp_xchg* x, const dcp_instance_view* v, const dcp_mla_args* a0,
                               void* stream) {
    DCP_REQUIRE(ctx && x && v && a0, DCP_E_INVALID_ARG, "NULL argument");
    DCP_REQUIRE(v->instance == x->cfg.self, DCP_E_INVALID_ARG, "view/instance mismatch");
    DCP_REQUIRE(v->n_rows <= x->cfg.n_max, DCP_E_SHAPE_OVERFLOW, "N %d > n_max %d", v->n_rows, x->cfg.n_max);
    DCP_REQUIRE(x->cfg.num_q_heads == mla::H && x->cfg.q_dim == mla::DK && x->cfg.o_dim == mla::DL &&
                    x->cfg.q_elem_bytes == 2,
                DCP_E_INVALID_ARG, "exchange pools must be MLA-shaped (128 heads, q_dim 576, o_dim 512, bf16 Q)");
    DCP_REQUIRE(a0->num_q_heads == mla::H && a0->kv_lora_rank == mla::DL && a0->rope_dim == mla::DR,
                DCP_E_UNSUPPORTED, "MLA shape");
    DCP_REQUIRE(a0->page_size == 16 || a0->page_size == 32 || a0->page_size == 64, DCP_E_UNSUPPORTED,
                "page_size %d (compiled: 16, 32, 64)", a0->page_size);
    DCP_REQUIRE(a0->kv_pool && a0->workspace && a0->num_frames > 0 && a0->num_frames < (int64_t(1) << 31),
                DCP_E_INVALID_ARG, "kv_pool / workspace / num_frames");
    DCP_REQUIRE((reinterpret_cast<uintptr_t>(a0->kv_pool) & 15) == 0, DCP_E_INVALID_ARG, "kv_pool alignment");
    // shard arrays from the view; grids sized for n_max shards (R is read on the device)
    dcp_mla_args a = *a0;
    a.num_shards = x->cfg.n_max;
    a.block_table = v->block_table;
    a.cu_pages = v->cu_pages;
    a.shard_len = v->shard_len;
    a.page_fill = v->page_fill;
    a.q = nullptr;
    a.out = nullptr;
    a.lse = nullptr;
    const size_t need = dcp_mla_workspace_bytes(ctx, a.num_shards);
    DCP_REQUIRE(a.workspace_bytes >= need, DCP_E_INVALID_ARG, "workspace %zu < %zu bytes (size it for n_max)",
                a.workspace_bytes, need);
    const MlaRoute rt{x, v};
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (a.page_size == 16) return mla_launch<16>(ctx, &a, s, &rt);
    if (a.page_size == 32) return mla_launch<32>(ctx, &a, s, &rt);
    return mla_launch<64>(ctx, &a, s, &rt);
}

}  // extern "C"
