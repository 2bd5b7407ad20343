// SPDX-License-Identifier: Apache-2.0
// C ABI: K4/K5 MoE dispatch / combine (dcp_capi.h).
#include <cstring>

#include "capi_common.cuh"
#include <cstdlib>
#include "moe.cuh"
#include "moe_internal.cuh"

using namespace dcp;


namespace {
size_t al(size_t x) { return (x + 255) & ~size_t(255); }
size_t dispatch_smem(const dcp_moe* x) { return (size_t)x->cfg.m_max * (x->cfg.world + 1) * 4; }
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
    DCP_REQUIRE(c->timeout_ms >= 0, DCP_E_INVALID_ARG, "timeout_ms");
    DCP_CUDA_TRY(cudaSetDevice(ctx->device));
    auto* x = new dcp_moe();
    x->ctx = ctx;
    x->cfg = *c;
    if (x->cfg.timeout_ms == 0) x->cfg.timeout_ms = 10000;
    const size_t W = c->world, H = c->hidden, m = c->m_max, meta = 2 + 2 * c->topk;
    MoePeers& h = x->host;
    h.sz_rx_x = al(W * m * H * 2);
    h.sz_rx_meta = al(W * m * meta * 4);
    h.sz_rx_cnt = al(W * 16);
    h.sz_rx_arr = al(W * 4);
    h.sz_cb_y = al(m * W * H * 2);
    h.sz_cb_arr = al(W * 4);
    size_t o = 0;
    h.off_rx_x = o;    o += 2 * h.sz_rx_x;
    h.off_rx_meta = o; o += 2 * h.sz_rx_meta;
    h.off_rx_cnt = o;  o += 2 * h.sz_rx_cnt;
    h.off_rx_arr = o;  o += 2 * h.sz_rx_arr;
    h.off_cb_y = o;    o += 2 * h.sz_cb_y;
    h.off_cb_arr = o;  o += 2 * h.sz_cb_arr;
    h.off_done = o;    o += 256;
    DCP_CUDA_TRY(cudaMalloc(&x->pool, o));
    DCP_CUDA_TRY(cudaMemset(x->pool, 0, o));
    size_t l = 0;
    const size_t o_ep = l;   l = al(l + 4);
    const size_t o_err = l;  l = al(l + 16);
    const size_t o_dev = l;  l = al(l + sizeof(MoePeers));
    const size_t o_slot = l; l = al(l + m * W * 4);
    const size_t o_cs = l;   l = al(l + 2 * W * 4);
    const size_t o_ct = l;   l = al(l + 2 * W * 4);
    const size_t o_cnt = l;  l = al(l + W * 4);
    const size_t o_off = l;  l = al(l + (W + 1) * 4);
    const size_t o_tk = l;   l = al(l + 4);
    DCP_CUDA_TRY(cudaMalloc(&x->local, l));
    DCP_CUDA_TRY(cudaMemset(x->local, 0, l));
    x->epoch = reinterpret_cast<uint32_t*>(x->local + o_ep);
    x->err = reinterpret_cast<uint32_t*>(x->local + o_err);
    x->dev = reinterpret_cast<MoePeers*>(x->local + o_dev);
    h.W = c->world;
    h.self = c->self;
    h.H = c->hidden;
    h.topk = c->topk;
    h.e_per_rank = c->num_experts / c->world;
    h.m_max = c->m_max;
    h.meta = (int32_t)meta;
    h.epoch = x->epoch;
    h.wc.err = x->err;
    h.wc.timeout_ns = static_cast<uint64_t>(x->cfg.timeout_ms) * 1000000ull;
    h.slot_tbl = reinterpret_cast<int32_t*>(x->local + o_slot);
    h.cum_sent = reinterpret_cast<uint32_t*>(x->local + o_cs);
    h.cb_target = reinterpret_cast<uint32_t*>(x->local + o_ct);
    h.counts = reinterpret_cast<int32_t*>(x->local + o_cnt);
    h.offs = reinterpret_cast<int32_t*>(x->local + o_off);
    h.exit_ticket = reinterpret_cast<int32_t*>(x->local + o_tk);
    // one wave of CTAs for K4 / K5b (a CTA per token / per received row beyond that)
    h.chunks = ctx->num_sms;
    h.base[c->self] = x->pool;
    const size_t sm = dispatch_smem(x);
    if (sm > 48 * 1024)
        DCP_CUDA_TRY(cudaFuncSetAttribute(moe_dispatch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(sm)));
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
    DCP_CUDA_TRY(cudaSetDevice(x->ctx->device));
    cudaIpcMemHandle_t h;
    std::memcpy(&h, h64, 64);
    void* base = nullptr;
    DCP_CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    x->opened[peer] = base;
    x->host.base[peer] = static_cast<char*>(base);
    return DCP_OK;
}

int dcp_moe_set_peer_local(dcp_moe* x, int32_t peer, const dcp_moe* other) {
    DCP_REQUIRE(x && other && peer >= 0 && peer < x->cfg.world, DCP_E_INVALID_ARG, "peer");
    DCP_REQUIRE(x->cfg.hidden == other->cfg.hidden && x->cfg.topk == other->cfg.topk &&
                    x->cfg.m_max == other->cfg.m_max && x->cfg.world == other->cfg.world &&
                    x->cfg.num_experts == other->cfg.num_experts,
                DCP_E_INVALID_ARG, "peer pool shapes differ");
    if (other->ctx->device != x->ctx->device) {
        cudaError_t e = cudaDeviceEnablePeerAccess(other->ctx->device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) {
            set_error("cudaDeviceEnablePeerAccess: %s", cudaGetErrorString(e));
            return DCP_E_CUDA;
        }
        cudaGetLastError();
    }
    x->host.base[peer] = other->pool;
    return DCP_OK;
}

int dcp_moe_commit(dcp_moe* x) {
    DCP_REQUIRE(x, DCP_E_INVALID_ARG, "NULL argument");
    for (int s = 0; s < x->cfg.world; ++s) DCP_REQUIRE(x->host.base[s], DCP_E_INVALID_ARG, "peer %d not set", s);
    DCP_CUDA_TRY(cudaMemcpy(x->dev, &x->host, sizeof(MoePeers), cudaMemcpyHostToDevice));
    x->committed = true;
    return DCP_OK;
}

int dcp_moe_begin_step(dcp_moe* x, void* stream) {
    DCP_REQUIRE(x && x->committed, DCP_E_INVALID_ARG, "NULL or uncommitted MoE exchange (dcp_moe_commit)");
    DCP_CUDA_TRY(launch_pdl(moe_begin_step_kernel, dim3(1), dim3(32), 0, static_cast<cudaStream_t>(stream), x->host));
    ++x->host_epoch;
    x->received = false;
    return DCP_OK;
}

int dcp_moe_status(dcp_moe* x, uint32_t* info) {
    DCP_REQUIRE(x, DCP_E_INVALID_ARG, "NULL argument");
    DCP_CUDA_TRY(cudaSetDevice(x->ctx->device));
    DCP_CUDA_TRY(cudaDeviceSynchronize());
    uint32_t e[4];
    DCP_CUDA_TRY(cudaMemcpy(e, x->err, sizeof(e), cudaMemcpyDeviceToHost));
    if (info) std::memcpy(info, e, sizeof(e));
    if (e[0] == XERR_NONE) return DCP_OK;
    DCP_CUDA_TRY(cudaMemset(x->err, 0, sizeof(e)));
    set_error("MoE exchange wait timed out: site %u peer %u row %u, wanted %u, saw %u", e[1] >> 24,
              (e[1] >> 16) & 0xff, e[1] & 0xffff, e[2], e[3]);
    return DCP_E_TIMEOUT;
}

int32_t dcp_moe_meta_width(const dcp_moe* x) { return x ? 2 + 2 * x->cfg.topk : 0; }

int32_t dcp_moe_parity(const dcp_moe* x) { return x ? static_cast<int32_t>(x->host_epoch & 1) : 0; }

int dcp_moe_regions(dcp_moe* x, int32_t parity, void** x_region, int32_t** meta_region) {
    DCP_REQUIRE(x && (parity == 0 || parity == 1), DCP_E_INVALID_ARG, "bad argument");
    if (x_region) *x_region = x->pool + x->host.off_rx_x + parity * x->host.sz_rx_x;
    if (meta_region)
        *meta_region = reinterpret_cast<int32_t*>(x->pool + x->host.off_rx_meta + parity * x->host.sz_rx_meta);
    return DCP_OK;
}

int dcp_moe_dispatch(dcp_moe* x, const void* x_local, const int32_t* idx, const float* w, const int32_t* m_count,
                     void* stream) {
    DCP_NVTX("K4 moe dispatch");
    // x_local / idx / w may be NULL when the instance has no MoE-bound tokens (M = 0)
    DCP_REQUIRE(x && m_count, DCP_E_INVALID_ARG, "NULL argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    x->m_count_dev = m_count;
    DCP_CUDA_TRY(launch_pdl(moe_dispatch_kernel, dim3(x->host.chunks), dim3(MOE_THREADS), dispatch_smem(x), s, x->host,
                            static_cast<const __nv_bfloat16*>(x_local), idx, w, m_count, 0, 0));
    return DCP_OK;
}

int dcp_moe_step_dispatch(dcp_moe* x, const void* x_local, const int32_t* idx, const float* w,
                          const int32_t* m_count, void* stream) {
    DCP_NVTX("K4 moe step dispatch");
    DCP_REQUIRE(x && x->committed && m_count, DCP_E_INVALID_ARG, "NULL or uncommitted MoE exchange");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    x->m_count_dev = m_count;
    DCP_CUDA_TRY(launch_pdl(moe_dispatch_kernel, dim3(x->host.chunks), dim3(MOE_THREADS), dispatch_smem(x), s, x->host,
                            static_cast<const __nv_bfloat16*>(x_local), idx, w, m_count, 1, 0));
    ++x->host_epoch;  // what dcp_moe_begin_step does on the host
    x->received = false;
    return DCP_OK;
}

int dcp_moe_step_dispatch_recv(dcp_moe* x, const void* x_local, const int32_t* idx, const float* w,
                               const int32_t* m_count, void* stream) {
    DCP_NVTX("K4+K5a moe step dispatch + receive (fused)");
    DCP_REQUIRE(x && x->committed && m_count, DCP_E_INVALID_ARG, "NULL or uncommitted MoE exchange");
    DCP_REQUIRE(MOE_SINGLE_RELEASE, DCP_E_UNSUPPORTED, "fused receive needs the single-release K4 build");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    x->m_count_dev = m_count;
    DCP_CUDA_TRY(launch_pdl(moe_dispatch_kernel, dim3(x->host.chunks), dim3(MOE_THREADS), dispatch_smem(x), s, x->host,
                            static_cast<const __nv_bfloat16*>(x_local), idx, w, m_count, 1, 1));
    ++x->host_epoch;
    x->received = true;  // the counts / offsets of dcp_moe_receive_regions are written by this launch
    return DCP_OK;
}

int dcp_moe_receive_regions(dcp_moe* x, void* stream) {
    DCP_NVTX("K5a moe receive");
    DCP_REQUIRE(x, DCP_E_INVALID_ARG, "NULL argument");
    DCP_CUDA_TRY(launch_pdl(moe_receive_counts_kernel, dim3(1), dim3(32), 0, static_cast<cudaStream_t>(stream), x->host));
    x->received = true;
    return DCP_OK;
}

int dcp_moe_receive_async(dcp_moe* x, void* x_rows, int32_t* meta_rows, void* stream) {
    DCP_REQUIRE(x && x_rows && meta_rows, DCP_E_INVALID_ARG, "NULL argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int rows = x->cfg.world * x->cfg.m_max;
    int grid = rows;  // up to one CTA per received row (warp groups per row, moe.cuh)
    if (grid > 4 * x->ctx->num_sms) grid = 4 * x->ctx->num_sms;
    DCP_CUDA_TRY(launch_pdl(moe_receive_compact_kernel, dim3(grid), dim3(256), 0, s, x->host,
                            static_cast<__nv_bfloat16*>(x_rows), meta_rows));
    x->received = true;
    return DCP_OK;
}

const int32_t* dcp_moe_recv_counts_dev(const dcp_moe* x) { return x ? x->host.counts : nullptr; }

int32_t dcp_moe_receive(dcp_moe* x, void* x_rows, int32_t* meta_rows, int32_t* counts, void* stream) {
    if (int rc = dcp_moe_receive_async(x, x_rows, meta_rows, stream)) return rc;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    int32_t c[PL_MAXW];
    DCP_CUDA_TRY(cudaMemcpyAsync(c, x->host.counts, x->cfg.world * 4, cudaMemcpyDeviceToHost, s));
    DCP_CUDA_TRY(cudaStreamSynchronize(s));
    int32_t R = 0;
    for (int i = 0; i < x->cfg.world; ++i) {
        if (counts) counts[i] = c[i];
        R += c[i];
    }
    return R;
}

static int combine_put(dcp_moe* x, const void* y, int region, void* stream) {
    DCP_REQUIRE(x && y && x->received, DCP_E_INVALID_ARG, "call a dcp_moe_receive* first");
    DCP_CUDA_TRY(launch_pdl(moe_combine_put_kernel, dim3(x->host.chunks), dim3(MOE_THREADS), 0,
                            static_cast<cudaStream_t>(stream), x->host, static_cast<const __nv_bfloat16*>(y), region));
    return DCP_OK;
}

int dcp_moe_combine_put(dcp_moe* x, const void* y_rows, void* stream) { return combine_put(x, y_rows, 0, stream); }

int dcp_moe_combine_put_regions(dcp_moe* x, const void* y_region, void* stream) {
    DCP_NVTX("K5b moe combine_put");
    return combine_put(x, y_region, 1, stream);
}

int dcp_moe_expert_identity(dcp_moe* x, void* y_region, void* stream) {
    DCP_REQUIRE(x && y_region && x->received, DCP_E_INVALID_ARG, "call dcp_moe_receive_regions first");
    int grid = (x->cfg.world * x->cfg.m_max + 7) / 8;
    if (grid > 2 * x->ctx->num_sms) grid = 2 * x->ctx->num_sms;
    DCP_CUDA_TRY(launch_pdl(moe_expert_identity_kernel, dim3(grid), dim3(256), 0, static_cast<cudaStream_t>(stream),
                            x->host, static_cast<__nv_bfloat16*>(y_region)));
    return DCP_OK;
}

int dcp_moe_combine_reduce(dcp_moe* x, float* out, void* stream) {
    DCP_NVTX("K5c moe combine_reduce");
    DCP_REQUIRE(x && out && x->m_count_dev, DCP_E_INVALID_ARG, "call dcp_moe_dispatch first");
    const int groups = x->cfg.hidden / 4;  // hidden % 8 == 0
    DCP_CUDA_TRY(launch_pdl(moe_combine_reduce_kernel, dim3(x->cfg.m_max, (groups + 255) / 256), dim3(256), 0,
                            static_cast<cudaStream_t>(stream), x->host, x->m_count_dev, out));
    return DCP_OK;
}

int dcp_moe_combine_fused(dcp_moe* x, const void* y_region, float* out, void* stream) {
    DCP_NVTX("K5b+K5c moe combine (fused)");
    DCP_REQUIRE(x && y_region && out && x->received && x->m_count_dev, DCP_E_INVALID_ARG,
                "call dcp_moe_dispatch and dcp_moe_receive_regions first");
    DCP_CUDA_TRY(launch_pdl(moe_combine_fused_kernel, dim3(x->host.chunks), dim3(MOE_THREADS), 0,
                            static_cast<cudaStream_t>(stream), x->host, static_cast<const __nv_bfloat16*>(y_region),
                            x->m_count_dev, out));
    return DCP_OK;
}

}  // extern "C"
