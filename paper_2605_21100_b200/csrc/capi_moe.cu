// SPDX-License-Identifier: Apache-2.0
// C ABI: K4/K5 MoE dispatch / combine (dcp_capi.h).
#include <cstring>

#include "capi_common.cuh"
#include <cstdlib>
#include "moe.cuh"

using namespace dcp;

struct dcp_moe {
    dcp_ctx* ctx = nullptr;
    dcp_moe_config cfg{};
    char* pool = nullptr;
    size_t off_x = 0, off_meta = 0, off_flag = 0, off_cnt = 0, off_cb = 0, off_cbf = 0;
    char* local = nullptr;
    MoePeers host{};
    MoePeers* dev = nullptr;
    uint32_t* epoch = nullptr;
    int32_t* slot_tbl = nullptr;
    int32_t* row_src = nullptr;
    int32_t* counts = nullptr;
    const int32_t* m_count_dev = nullptr;
    const int32_t* meta_rows = nullptr;
    void* opened[PL_MAXW] = {};
};

namespace {
size_t al(size_t x) { return (x + 255) & ~size_t(255); }
void fill(dcp_moe* x, int peer, char* base) {
    x->host.rx_x[peer] = reinterpret_cast<__nv_bfloat16*>(base + x->off_x);
    x->host.rx_meta[peer] = reinterpret_cast<int32_t*>(base + x->off_meta);
    x->host.rx_flag[peer] = reinterpret_cast<uint32_t*>(base + x->off_flag);
    x->host.rx_count[peer] = reinterpret_cast<int32_t*>(base + x->off_cnt);
    x->host.cb_y[peer] = reinterpret_cast<__nv_bfloat16*>(base + x->off_cb);
    x->host.cb_flag[peer] = reinterpret_cast<uint32_t*>(base + x->off_cbf);
}
}  // namespace

extern "C" {

int dcp_moe_create(dcp_ctx* ctx, const dcp_moe_config* c, dcp_moe** out) {
    DCP_REQUIRE(ctx && c && out, DCP_E_INVALID_ARG, "NULL argument");
    DCP_REQUIRE(c->world >= 1 && c->world <= PL_MAXW && c->self >= 0 && c->self < c->world, DCP_E_INVALID_ARG,
                "world/self");
    DCP_REQUIRE(c->hidden > 0 && c->hidden % 8 == 0, DCP_E_UNSUPPORTED, "hidden %d (multiple of 8)", c->hidden);
    DCP_REQUIRE(c->topk >= 1 && c->topk <= MOE_MAXK, DCP_E_UNSUPPORTED, "topk %d", c->topk);
    DCP_REQUIRE(c->num_experts >= c->world && c->num_experts % c->world == 0, DCP_E_CONFIG,
                "num_experts must be a multiple of world");
    DCP_REQUIRE(c->m_max >= 1 && c->m_max <= 1024, DCP_E_UNSUPPORTED, "m_max %d (<= 1024)", c->m_max);
    DCP_CUDA_TRY(cudaSetDevice(ctx->device));
    auto* x = new dcp_moe();
    x->ctx = ctx;
    x->cfg = *c;
    const size_t W = c->world, H = c->hidden, m = c->m_max, meta = 2 + 2 * c->topk;
    size_t o = 0;
    x->off_x = o;    o = al(o + W * m * H * 2);
    x->off_meta = o; o = al(o + W * m * meta * 4);
    x->off_flag = o; o = al(o + W * 4);
    x->off_cnt = o;  o = al(o + W * 4);
    x->off_cb = o;   o = al(o + m * W * H * 2);
    x->off_cbf = o;  o = al(o + W * 4);
    DCP_CUDA_TRY(cudaMalloc(&x->pool, o));
    DCP_CUDA_TRY(cudaMemset(x->pool, 0, o));
    size_t l = 0;
    const size_t o_ep = l;   l = al(l + 4);
    const size_t o_dev = l;  l = al(l + sizeof(MoePeers));
    const size_t o_slot = l; l = al(l + m * W * 4);
    const size_t o_src = l;  l = al(l + W * m * 4);
    const size_t o_cnt = l;  l = al(l + W * 4);
    const size_t o_dd = l;   l = al(l + W * 4);
    const size_t o_cd = l;   l = al(l + W * 4);
    DCP_CUDA_TRY(cudaMalloc(&x->local, l));
    DCP_CUDA_TRY(cudaMemset(x->local, 0, l));
    x->epoch = reinterpret_cast<uint32_t*>(x->local + o_ep);
    x->dev = reinterpret_cast<MoePeers*>(x->local + o_dev);
    x->slot_tbl = reinterpret_cast<int32_t*>(x->local + o_slot);
    x->row_src = reinterpret_cast<int32_t*>(x->local + o_src);
    x->counts = reinterpret_cast<int32_t*>(x->local + o_cnt);
    x->host.W = c->world;
    x->host.self = c->self;
    x->host.H = c->hidden;
    x->host.topk = c->topk;
    x->host.e_per_rank = c->num_experts / c->world;
    x->host.m_max = c->m_max;
    x->host.meta = (int32_t)meta;
    x->host.epoch = x->epoch;
    x->host.disp_done = reinterpret_cast<int32_t*>(x->local + o_dd);
    x->host.cb_done = reinterpret_cast<int32_t*>(x->local + o_cd);
    static const int max_chunks = [] { const char* e = std::getenv("DCP_MOE_CHUNKS"); return e ? std::atoi(e) : 128; }();
    x->host.chunks = static_cast<int32_t>(m < max_chunks ? m : max_chunks);
    fill(x, c->self, x->pool);
    *out = x;
    return DCP_OK;
}

int dcp_moe_destroy(dcp_moe* x) {
    if (!x) return DCP_OK;
    for (int i = 0; i < PL_MAXW; ++i)
        if (x->opened[i]) cudaIpcCloseMemHandle(x->opened[i]);
    cudaFree(x->pool);
    cudaFree(x->local);
    delete x;
    return DCP_OK;
}

int dcp_moe_ipc_handle(dcp_moe* x, void* h64) {
    DCP_REQUIRE(x && h64, DCP_E_INVALID_ARG, "NULL argument");
    cudaIpcMemHandle_t h;
    DCP_CUDA_TRY(cudaIpcGetMemHandle(&h, x->pool));
    std::memcpy(h64, &h, 64);
    return DCP_OK;
}

int dcp_moe_open_peer_ipc(dcp_moe* x, int32_t peer, const void* h64) {
    DCP_REQUIRE(x && h64 && peer >= 0 && peer < x->cfg.world && peer != x->cfg.self, DCP_E_INVALID_ARG, "peer");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, h64, 64);
    void* base = nullptr;
    DCP_CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    x->opened[peer] = base;
    fill(x, peer, static_cast<char*>(base));
    return DCP_OK;
}

int dcp_moe_set_peer_local(dcp_moe* x, int32_t peer, const dcp_moe* other) {
    DCP_REQUIRE(x && other && peer >= 0 && peer < x->cfg.world, DCP_E_INVALID_ARG, "peer");
    DCP_REQUIRE(x->cfg.hidden == other->cfg.hidden && x->cfg.topk == other->cfg.topk &&
                    x->cfg.m_max == other->cfg.m_max && x->cfg.world == other->cfg.world,
                DCP_E_INVALID_ARG, "peer pool shapes differ");
    if (other->ctx->device != x->ctx->device) {
        cudaError_t e = cudaDeviceEnablePeerAccess(other->ctx->device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
            set_error("cudaDeviceEnablePeerAccess: %s", cudaGetErrorString(e));
            return DCP_E_CUDA;
        }
        cudaGetLastError();
    }
    fill(x, peer, other->pool);
    return DCP_OK;
}

int dcp_moe_commit(dcp_moe* x) {
    DCP_REQUIRE(x, DCP_E_INVALID_ARG, "NULL argument");
    for (int s = 0; s < x->cfg.world; ++s) DCP_REQUIRE(x->host.rx_x[s], DCP_E_INVALID_ARG, "peer %d not set", s);
    DCP_CUDA_TRY(cudaMemcpy(x->dev, &x->host, sizeof(MoePeers), cudaMemcpyHostToDevice));
    return DCP_OK;
}

int dcp_moe_begin_step(dcp_moe* x, void* stream) {
    DCP_REQUIRE(x, DCP_E_INVALID_ARG, "NULL argument");
    epoch_bump_kernel_moe<<<1, 1, 0, static_cast<cudaStream_t>(stream)>>>(x->epoch);
    DCP_CUDA_TRY(cudaGetLastError());
    return DCP_OK;
}

int32_t dcp_moe_meta_width(const dcp_moe* x) { return x ? 2 + 2 * x->cfg.topk : 0; }

int dcp_moe_dispatch(dcp_moe* x, const void* x_local, const int32_t* idx, const float* w, const int32_t* m_count,
                     void* stream) {
    // x_local / idx / w may be NULL when the instance has no MoE-bound tokens (M = 0)
    DCP_REQUIRE(x && m_count, DCP_E_INVALID_ARG, "NULL argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    x->m_count_dev = m_count;
    moe_dispatch_kernel<<<dim3(x->host.chunks, x->cfg.world), 128, 0, s>>>(
        x->dev, static_cast<const __nv_bfloat16*>(x_local), idx, w, m_count, x->slot_tbl);
    DCP_CUDA_TRY(cudaGetLastError());
    return DCP_OK;
}

int dcp_moe_receive_async(dcp_moe* x, void* x_rows, int32_t* meta_rows, void* stream) {
    DCP_REQUIRE(x && x_rows && meta_rows, DCP_E_INVALID_ARG, "NULL argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int rows = x->cfg.world * x->cfg.m_max;
    int grid = rows;  // up to one CTA per received row (warp groups per row, moe.cuh)
    if (grid > 4 * x->ctx->num_sms) grid = 4 * x->ctx->num_sms;
    moe_receive_kernel<<<grid, 256, 0, s>>>(x->dev, static_cast<__nv_bfloat16*>(x_rows), meta_rows, x->row_src,
                                            x->counts);
    DCP_CUDA_TRY(cudaGetLastError());
    x->meta_rows = meta_rows;
    return DCP_OK;
}

const int32_t* dcp_moe_recv_counts_dev(const dcp_moe* x) { return x ? x->counts : nullptr; }

int32_t dcp_moe_receive(dcp_moe* x, void* x_rows, int32_t* meta_rows, int32_t* counts, void* stream) {
    DCP_REQUIRE(x && x_rows && meta_rows, DCP_E_INVALID_ARG, "NULL argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // one CTA per received row, at most W * m_max rows
    const int rows = x->cfg.world * x->cfg.m_max;
    int grid = rows;  // up to one CTA per received row (warp groups per row, moe.cuh)
    if (grid > 4 * x->ctx->num_sms) grid = 4 * x->ctx->num_sms;
    moe_receive_kernel<<<grid, 256, 0, s>>>(x->dev, static_cast<__nv_bfloat16*>(x_rows), meta_rows, x->row_src,
                                            x->counts);
    DCP_CUDA_TRY(cudaGetLastError());
    x->meta_rows = meta_rows;
    int32_t c[PL_MAXW];
    DCP_CUDA_TRY(cudaMemcpyAsync(c, x->counts, x->cfg.world * 4, cudaMemcpyDeviceToHost, s));
    DCP_CUDA_TRY(cudaStreamSynchronize(s));
    int32_t R = 0;
    for (int i = 0; i < x->cfg.world; ++i) {
        if (counts) counts[i] = c[i];
        R += c[i];
    }
    return R;
}

int dcp_moe_combine_put(dcp_moe* x, const void* y_rows, void* stream) {
    DCP_REQUIRE(x && y_rows && x->meta_rows, DCP_E_INVALID_ARG, "call dcp_moe_receive first");
    moe_combine_put_kernel<<<dim3(x->host.chunks, x->cfg.world), 128, 0, static_cast<cudaStream_t>(stream)>>>(
        x->dev, static_cast<const __nv_bfloat16*>(y_rows), x->meta_rows, x->counts);
    DCP_CUDA_TRY(cudaGetLastError());
    return DCP_OK;
}

int dcp_moe_combine_reduce(dcp_moe* x, float* out, void* stream) {
    DCP_REQUIRE(x && out && x->m_count_dev, DCP_E_INVALID_ARG, "call dcp_moe_dispatch first");
    const int groups = x->cfg.hidden / 4;  // hidden % 8 == 0
    moe_combine_reduce_kernel<<<dim3(x->cfg.m_max, (groups + 255) / 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        x->dev, x->m_count_dev, x->slot_tbl, out);
    DCP_CUDA_TRY(cudaGetLastError());
    return DCP_OK;
}

}  // extern "C"
