// SPDX-License-Identifier: Apache-2.0
// C ABI: the routing-based exchange (K2 Q-route, K3 LSE merge) — dcp_capi.h.
#include <algorithm>
#include <cstring>

#include "exchange_kernels.cuh"
#include "xchg_internal.cuh"

using namespace dcp;

namespace {

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

}  // namespace

namespace dcp {
int xchg_route_q_grid(dcp_xchg* x, const dcp_instance_view* v, int grid, cudaStream_t s) {
    q_route_put_kernel<<<grid, 128, 0, s>>>(x->host, x->q_local, v->m_count_all, v->m_nrow);
    DCP_CUDA_TRY(cudaGetLastError());
    return DCP_OK;
}
int xchg_merge_grid(dcp_xchg* x, const dcp_instance_view* v, int grid, cudaStream_t s) {
    lse_merge_kernel<<<grid, 128, 0, s>>>(x->host, v->m_count_all, v->m_k, v->m_kv, x->out, x->out_lse);
    DCP_CUDA_TRY(cudaGetLastError());
    return DCP_OK;
}
}  // namespace dcp

extern "C" {

int dcp_xchg_create(dcp_ctx* ctx, const dcp_xchg_config* c0, dcp_xchg** out) {
    DCP_REQUIRE(ctx && c0 && out, DCP_E_INVALID_ARG, "NULL argument");
    dcp_xchg_config c = *c0;
    if (c.q_dim == 0) c.q_dim = c.head_dim;
    if (c.o_dim == 0) c.o_dim = c.head_dim;
    if (c.q_elem_bytes == 0) c.q_elem_bytes = 2;
    if (c.timeout_ms == 0) c.timeout_ms = 10000;
    DCP_REQUIRE(c.world >= 1 && c.world <= PL_MAXW, DCP_E_UNSUPPORTED, "world %d", c.world);
    DCP_REQUIRE(c.self >= 0 && c.self < c.world, DCP_E_INVALID_ARG, "self %d", c.self);
    DCP_REQUIRE(c.num_q_heads > 0 && c.q_dim > 0 && c.o_dim > 0 && c.o_dim % 32 == 0, DCP_E_UNSUPPORTED,
                "o_dim %d (multiple of 32)", c.o_dim);
    DCP_REQUIRE(c.q_elem_bytes == 2 || c.q_elem_bytes == 4, DCP_E_UNSUPPORTED, "q_elem_bytes %d", c.q_elem_bytes);
    DCP_REQUIRE((size_t)c.num_q_heads * c.q_dim * c.q_elem_bytes % 16 == 0, DCP_E_UNSUPPORTED,
                "query rows must be a multiple of 16 bytes");
    DCP_REQUIRE(c.n_max > 0 && c.m_max > 0, DCP_E_INVALID_ARG, "n_max/m_max");
    DCP_REQUIRE(c.timeout_ms > 0, DCP_E_INVALID_ARG, "timeout_ms");
    DCP_CUDA_TRY(cudaSetDevice(ctx->device));
    auto* x = new dcp_xchg();
    x->ctx = ctx;
    x->cfg = c;
    const size_t W = c.world, hq = c.num_q_heads, n = c.n_max, m = c.m_max;
    const size_t qrow = hq * c.q_dim * c.q_elem_bytes;
    XchgPeers& h = x->host;
    h.sz_qrecv = align256(n * qrow);
    h.sz_qflag = align256(n * 4);
    h.sz_res_o = align256(m * W * hq * c.o_dim * 4);
    h.sz_res_lse = align256(m * W * hq * 4);
    h.sz_res_flag = align256(m * W * 4);
    size_t o = 0;
    h.off_qrecv = o;    o += 2 * h.sz_qrecv;
    h.off_qflag = o;    o += 2 * h.sz_qflag;
    h.off_res_o = o;    o += 2 * h.sz_res_o;
    h.off_res_lse = o;  o += 2 * h.sz_res_lse;
    h.off_res_flag = o; o += 2 * h.sz_res_flag;
    h.off_done = o;     o += 256;
    x->pool_bytes = o;
    DCP_CUDA_TRY(cudaMalloc(&x->pool, x->pool_bytes));
    DCP_CUDA_TRY(cudaMemset(x->pool, 0, x->pool_bytes));
    size_t lb = 0;
    const size_t off_q = lb;   lb = align256(lb + m * qrow);
    const size_t off_out = lb; lb = align256(lb + m * hq * c.o_dim * 4);
    const size_t off_lse = lb; lb = align256(lb + m * hq * 4);
    const size_t off_ep = lb;  lb = align256(lb + 4);
    const size_t off_err = lb; lb = align256(lb + 16);
    const size_t off_tk = lb;  lb = align256(lb + 4);
    const size_t off_dev = lb; lb = align256(lb + sizeof(XchgPeers));
    DCP_CUDA_TRY(cudaMalloc(&x->local, lb));
    DCP_CUDA_TRY(cudaMemset(x->local, 0, lb));
    x->q_local = x->local + off_q;
    x->out = reinterpret_cast<float*>(x->local + off_out);
    x->out_lse = reinterpret_cast<float*>(x->local + off_lse);
    x->epoch = reinterpret_cast<uint32_t*>(x->local + off_ep);
    x->err = reinterpret_cast<uint32_t*>(x->local + off_err);
    x->exit_ticket = reinterpret_cast<int32_t*>(x->local + off_tk);
    x->dev = reinterpret_cast<XchgPeers*>(x->local + off_dev);
    h.W = c.world;
    h.self = c.self;
    h.hq = c.num_q_heads;
    h.q_dim = c.q_dim;
    h.o_dim = c.o_dim;
    h.q_bytes = c.q_elem_bytes;
    h.n_max = c.n_max;
    h.m_max = c.m_max;
    h.epoch = x->epoch;
    h.wc.err = x->err;
    h.wc.timeout_ns = static_cast<uint64_t>(c.timeout_ms) * 1000000ull;
    h.base[c.self] = x->pool;
    *out = x;
    return DCP_OK;
}

int dcp_xchg_destroy(dcp_xchg* x) {
    if (!x) return DCP_OK;
    for (int i = 0; i < PL_MAXW; ++i)
        if (x->opened[i]) cudaIpcCloseMemHandle(x->opened[i]);
    cudaFree(x->pool);
    cudaFree(x->local);
    delete x;
    return DCP_OK;
}

int dcp_xchg_ipc_handle(dcp_xchg* x, void* handle64) {
    DCP_REQUIRE(x && handle64, DCP_E_INVALID_ARG, "NULL argument");
    cudaIpcMemHandle_t h;
    DCP_CUDA_TRY(cudaIpcGetMemHandle(&h, x->pool));
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(handle64, &h, 64);
    return DCP_OK;
}

int dcp_xchg_open_peer_ipc(dcp_xchg* x, int32_t peer, const void* handle64) {
    DCP_REQUIRE(x && handle64, DCP_E_INVALID_ARG, "NULL argument");
    DCP_REQUIRE(peer >= 0 && peer < x->cfg.world && peer != x->cfg.self, DCP_E_INVALID_ARG, "peer %d", peer);
    DCP_CUDA_TRY(cudaSetDevice(x->ctx->device));
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle64, 64);
    void* base = nullptr;
    DCP_CUDA_TRY(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    x->opened[peer] = base;
    x->host.base[peer] = static_cast<char*>(base);
    return DCP_OK;
}

int dcp_xchg_set_peer_local(dcp_xchg* x, int32_t peer, const dcp_xchg* other) {
    DCP_REQUIRE(x && other, DCP_E_INVALID_ARG, "NULL argument");
    DCP_REQUIRE(peer >= 0 && peer < x->cfg.world, DCP_E_INVALID_ARG, "peer %d", peer);
    DCP_REQUIRE(x->cfg.num_q_heads == other->cfg.num_q_heads && x->cfg.n_max == other->cfg.n_max &&
                    x->cfg.m_max == other->cfg.m_max && x->cfg.q_dim == other->cfg.q_dim &&
                    x->cfg.o_dim == other->cfg.o_dim && x->cfg.q_elem_bytes == other->cfg.q_elem_bytes &&
                    x->cfg.world == other->cfg.world,
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

int dcp_xchg_commit(dcp_xchg* x) {
    DCP_REQUIRE(x, DCP_E_INVALID_ARG, "NULL argument");
    for (int s = 0; s < x->cfg.world; ++s)
        DCP_REQUIRE(x->host.base[s] != nullptr, DCP_E_INVALID_ARG, "peer %d not set", s);
    DCP_CUDA_TRY(cudaMemcpy(x->dev, &x->host, sizeof(XchgPeers), cudaMemcpyHostToDevice));
    x->committed = true;
    return DCP_OK;
}

int dcp_xchg_begin_step(dcp_xchg* x, void* stream) {
    DCP_REQUIRE(x && x->committed, DCP_E_INVALID_ARG, "NULL or uncommitted exchange (dcp_xchg_commit)");
    xchg_begin_step_kernel<<<1, 32, 0, static_cast<cudaStream_t>(stream)>>>(x->host);
    DCP_CUDA_TRY(cudaGetLastError());
    return DCP_OK;
}

int dcp_xchg_status(dcp_xchg* x, uint32_t* info) {
    DCP_REQUIRE(x, DCP_E_INVALID_ARG, "NULL argument");
    DCP_CUDA_TRY(cudaSetDevice(x->ctx->device));
    DCP_CUDA_TRY(cudaDeviceSynchronize());
    uint32_t e[4];
    DCP_CUDA_TRY(cudaMemcpy(e, x->err, sizeof(e), cudaMemcpyDeviceToHost));
    if (info) std::memcpy(info, e, sizeof(e));
    if (e[0] == XERR_NONE) return DCP_OK;
    DCP_CUDA_TRY(cudaMemset(x->err, 0, sizeof(e)));
    set_error("exchange flag wait timed out: site %u peer %u row %u, wanted %u, saw %u", e[1] >> 24,
              (e[1] >> 16) & 0xff, e[1] & 0xffff, e[2], e[3]);
    return DCP_E_TIMEOUT;
}

int dcp_xchg_buffers(dcp_xchg* x, void** q_local, void** q_recv, float** out, float** out_lse) {
    DCP_REQUIRE(x, DCP_E_INVALID_ARG, "NULL argument");
    if (q_local) *q_local = x->q_local;
    if (q_recv) *q_recv = x->pool + x->host.off_qrecv;  // parity 0
    if (out) *out = x->out;
    if (out_lse) *out_lse = x->out_lse;
    return DCP_OK;
}

int dcp_xchg_write_queries(dcp_xchg* x, const void* q_rows, int32_t rows, void* stream) {
    DCP_REQUIRE(x && (rows == 0 || q_rows), DCP_E_INVALID_ARG, "NULL argument");
    DCP_REQUIRE(rows >= 0 && rows <= x->cfg.m_max, DCP_E_SHAPE_OVERFLOW, "rows %d > m_max %d", rows,
                x->cfg.m_max);
    const size_t bytes = (size_t)rows * x->cfg.num_q_heads * x->cfg.q_dim * x->cfg.q_elem_bytes;
    if (bytes)
        DCP_CUDA_TRY(cudaMemcpyAsync(x->q_local, q_rows, bytes, cudaMemcpyDeviceToDevice,
                                     static_cast<cudaStream_t>(stream)));
    return DCP_OK;
}

int dcp_route_q(dcp_xchg* x, const dcp_instance_view* v, void* stream) {
    DCP_NVTX("K2 q_route");
    DCP_REQUIRE(x && v, DCP_E_INVALID_ARG, "NULL argument");
    DCP_REQUIRE(v->instance == x->cfg.self && v->world == x->cfg.world, DCP_E_INVALID_ARG,
                "view of instance %d used on instance %d", v->instance, x->cfg.self);
    // rows beyond the pools would never be put and the receivers would wait forever
    DCP_REQUIRE(v->m_rows <= x->cfg.m_max && v->n_rows <= x->cfg.n_max, DCP_E_SHAPE_OVERFLOW,
                "execution shape (%d,%d) exceeds the exchange pools (%d,%d)", v->m_rows, v->n_rows, x->cfg.m_max,
                x->cfg.n_max);
    q_route_put_kernel<<<x->cfg.m_max, 128, 0, static_cast<cudaStream_t>(stream)>>>(x->host, x->q_local,
                                                                                  v->m_count_all, v->m_nrow);
    DCP_CUDA_TRY(cudaGetLastError());
    return DCP_OK;
}

int dcp_merge_partials(dcp_xchg* x, const dcp_instance_view* v, void* stream) {
    DCP_NVTX("K3 lse_merge");
    DCP_REQUIRE(x && v, DCP_E_INVALID_ARG, "NULL argument");
    DCP_REQUIRE(v->instance == x->cfg.self, DCP_E_INVALID_ARG, "view/instance mismatch");
    DCP_REQUIRE(v->m_rows <= x->cfg.m_max, DCP_E_SHAPE_OVERFLOW, "M %d > m_max %d", v->m_rows, x->cfg.m_max);
    lse_merge_kernel<<<x->cfg.m_max, 128, 0, static_cast<cudaStream_t>(stream)>>>(
        x->host, v->m_count_all, v->m_k, v->m_kv, x->out, x->out_lse);
    DCP_CUDA_TRY(cudaGetLastError());
    return DCP_OK;
}

struct dcp_step_graph {
    int m_hat[6] = {8, 16, 32, 64, 128, 256};
    int m_max = 0, n_max = 0;
    cudaGraphExec_t exec[6] = {};
    cudaGraph_t graph[6] = {};
};

int dcp_step_graph_create(dcp_ctx* ctx, dcp_xchg* x, const dcp_instance_view* v, const dcp_attn_args* a,
                          dcp_step_graph** out) {
    DCP_REQUIRE(ctx && x && v && a && out, DCP_E_INVALID_ARG, "NULL argument");
    DCP_REQUIRE(v->instance == x->cfg.self, DCP_E_INVALID_ARG, "view/instance mismatch");
    int rc = dcp_attn_prepare(ctx, a->num_kv_heads, a->num_q_heads / a->num_kv_heads, a->page_size);
    if (rc) return rc;
    cudaStream_t cs;
    DCP_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    auto* g = new dcp_step_graph();
    g->m_max = x->cfg.m_max;
    g->n_max = x->cfg.n_max;
    for (int i = 0; i < 6; ++i) {
        const int mh = std::min(g->m_hat[i], x->cfg.m_max);
        cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
        if (e == cudaSuccess) {
            xchg_begin_step_kernel<<<1, 32, 0, cs>>>(x->host);
            q_route_put_kernel<<<mh, 128, 0, cs>>>(x->host, x->q_local, v->m_count_all, v->m_nrow);
            rc = dcp_decode_attn_routed(ctx, x, v, a, cs);
            lse_merge_kernel<<<mh, 128, 0, cs>>>(x->host, v->m_count_all, v->m_k, v->m_kv, x->out, x->out_lse);
            e = cudaStreamEndCapture(cs, &g->graph[i]);
        }
        if (e == cudaSuccess && rc == 0) e = cudaGraphInstantiate(&g->exec[i], g->graph[i], 0);
        if (e != cudaSuccess || rc) {
            dcp_step_graph_destroy(g);
            cudaStreamDestroy(cs);
            if (rc) return rc;
            set_error("graph capture: %s", cudaGetErrorString(e));
            return DCP_E_CUDA;
        }
    }
    cudaStreamDestroy(cs);
    *out = g;
    return DCP_OK;
}

int dcp_step_graph_launch(dcp_step_graph* g, int32_t m, int32_t n, void* stream) {
    DCP_NVTX("step graph replay");
    DCP_REQUIRE(g, DCP_E_INVALID_ARG, "NULL graph");
    DCP_REQUIRE(m <= 256 && n <= 512 && m >= 0 && n >= 0, DCP_E_SHAPE_OVERFLOW,
                "execution shape (%d,%d) exceeds (256,512)", m, n);
    DCP_REQUIRE(m <= g->m_max && n <= g->n_max, DCP_E_SHAPE_OVERFLOW, "execution shape (%d,%d) exceeds the pools",
                m, n);
    int i = 0;
    while (g->m_hat[i] < m) ++i;  // bucket_shape: first dominating M^ (N^ shares the graph)
    DCP_CUDA_TRY(cudaGraphLaunch(g->exec[i], static_cast<cudaStream_t>(stream)));
    return DCP_OK;
}

int dcp_step_graph_count(const dcp_step_graph* g, int32_t* buckets) {
    if (buckets) *buckets = 48;
    return g ? 6 : 0;
}

int dcp_step_graph_destroy(dcp_step_graph* g) {
    if (!g) return DCP_OK;
    for (int i = 0; i < 6; ++i) {
        if (g->exec[i]) cudaGraphExecDestroy(g->exec[i]);
        if (g->graph[i]) cudaGraphDestroy(g->graph[i]);
    }
    delete g;
    return DCP_OK;
}

}  // extern "C"
