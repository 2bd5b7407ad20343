// SPDX-License-Identifier: Apache-2.0
// C ABI: whole-layer AOT decode graphs (dcp_layer_graph_*, dcp_capi.h) — PAPER.md Alg. 2
// (805-840) extended from the attention sub-step to the whole decode layer of one instance:
//
//   [K7 routing build] -> begin_step -> K2 Q-route -> K1 (+ Res-route) -> K3 merge
//     -> MoE begin_step -> K4 dispatch -> K5a receive (regions) -> expert stage
//     -> K5b combine_put -> K5c combine_reduce
//
// One executable graph per (M-bucket, MoE parity).  Every per-step quantity the kernels need
// (M / N counts, block tables, routes, epochs) is read from device memory K7 wrote, so a replay
// needs no metadata copy; the M-bucket only sizes the K2 / K3 grids (the kernels stride over
// the device M count, so any bucket is correct).  The expert stage is the caller's: a callback
// that enqueues its work (library GEMMs) on the capture stream, given the region pointers of
// the graph's parity — hence two graphs per bucket.  NULL selects the built-in gate-weighted
// identity expert (dcp_moe_expert_identity).
#include <vector>

#include "capi_common.cuh"
#include "moe_internal.cuh"
#include "planner_internal.cuh"
#include "xchg_internal.cuh"

using namespace dcp;

struct dcp_layer_graph {
    dcp_ctx* ctx = nullptr;
    dcp_layer_graph_desc d{};
    dcp_instance_view view{};           // copied: the graphs hold its device pointers
    dcp_attn_args attn{};
    std::vector<int> m_hat;
    std::vector<cudaGraph_t> graph;     // [parity][bucket]
    std::vector<cudaGraphExec_t> exec;
    uint64_t planner_gen = 0;
    int captures = 0;
};

namespace {

void release(dcp_layer_graph* g) {
    for (auto e : g->exec)
        if (e) cudaGraphExecDestroy(e);
    for (auto h : g->graph)
        if (h) cudaGraphDestroy(h);
    g->exec.clear();
    g->graph.clear();
}

// The layer, enqueued on `s` for the step whose MoE parity is `parity` (captured, never run eagerly).
int enqueue_layer(dcp_layer_graph* g, int mh, int parity, cudaStream_t s) {
    const dcp_layer_graph_desc& d = g->d;
    int rc = DCP_OK;
    if (d.planner) {
        dcp_planner* pl = d.planner;
        cudaStream_t keep = pl->stream;  // build_routing adopts its stream; the capture stream dies
        rc = dcp_planner_build_routing(pl, s);
        pl->stream = keep;
        if (rc) return rc;
    }
    if (d.fused_step) {
        if ((rc = dcp_decode_step_fused(g->ctx, d.xchg, &g->view, &g->attn, s))) return rc;
    } else {
        if ((rc = dcp_xchg_begin_step(d.xchg, s))) return rc;
        if ((rc = xchg_route_q_grid(d.xchg, &g->view, mh, s))) return rc;
        if ((rc = dcp_decode_attn_routed(g->ctx, d.xchg, &g->view, &g->attn, s))) return rc;
        if ((rc = xchg_merge_grid(d.xchg, &g->view, mh, s))) return rc;
    }
    if (!d.moe) return DCP_OK;
    dcp_moe* m = d.moe;
    if (d.fused_step) {  // one instance per process / GPU: K4 + K5a in one launch
        if ((rc = dcp_moe_step_dispatch_recv(m, d.moe_x, d.topk_idx, d.topk_w,
                                             g->view.m_count_all + g->view.instance, s)))
            return rc;
    } else {
        if ((rc = dcp_moe_step_dispatch(m, d.moe_x, d.topk_idx, d.topk_w, g->view.m_count_all + g->view.instance, s)))
            return rc;
        if ((rc = dcp_moe_receive_regions(m, s))) return rc;
    }
    if (d.expert) {
        void* xr = nullptr;
        int32_t* mr = nullptr;
        if ((rc = dcp_moe_regions(m, parity, &xr, &mr))) return rc;
        d.expert(d.expert_user, s, parity, xr, mr, dcp_moe_recv_counts_dev(m), d.y_region);
        DCP_CUDA_TRY(cudaGetLastError());
    } else if ((rc = dcp_moe_expert_identity(m, d.y_region, s))) {
        return rc;
    }
    // one instance per process / GPU (the fused step's condition): K5b + K5c in one launch
    if (d.fused_step) return dcp_moe_combine_fused(m, d.y_region, d.moe_out, s);
    if ((rc = dcp_moe_combine_put_regions(m, d.y_region, s))) return rc;
    return dcp_moe_combine_reduce(m, d.moe_out, s);
}

int capture_all(dcp_layer_graph* g) {
    release(g);
    const int nb = static_cast<int>(g->m_hat.size());
    g->graph.assign(2 * nb, nullptr);
    g->exec.assign(2 * nb, nullptr);
    int rc = dcp_attn_prepare(g->ctx, g->attn.num_kv_heads, g->attn.num_q_heads / g->attn.num_kv_heads,
                              g->attn.page_size);
    if (rc) return rc;
    // host mirrors the capture must not disturb
    const uint32_t moe_epoch = g->d.moe ? g->d.moe->host_epoch : 0;
    const bool moe_received = g->d.moe ? g->d.moe->received : false;
    const int32_t* moe_mcount = g->d.moe ? g->d.moe->m_count_dev : nullptr;
    const bool routing_valid = g->d.planner ? g->d.planner->routing_valid : false;
    cudaStream_t cs;
    DCP_CUDA_TRY(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    for (int par = 0; par < 2 && rc == DCP_OK; ++par) {
        for (int i = 0; i < nb && rc == DCP_OK; ++i) {
            const int k = par * nb + i;
            cudaError_t e = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
            if (e != cudaSuccess) {
                set_error("cudaStreamBeginCapture: %s", cudaGetErrorString(e));
                rc = DCP_E_CUDA;
                break;
            }
            rc = enqueue_layer(g, g->m_hat[i], par, cs);
            e = cudaStreamEndCapture(cs, &g->graph[k]);
            if (rc == DCP_OK && e == cudaSuccess) e = cudaGraphInstantiate(&g->exec[k], g->graph[k], 0);
            if (rc == DCP_OK && e != cudaSuccess) {
                set_error("layer graph capture: %s", cudaGetErrorString(e));
                rc = DCP_E_CUDA;
            }
        }
    }
    cudaStreamDestroy(cs);
    if (g->d.moe) {
        g->d.moe->host_epoch = moe_epoch;
        g->d.moe->received = moe_received;
        g->d.moe->m_count_dev = moe_mcount;
    }
    if (g->d.planner) {
        g->d.planner->routing_valid = routing_valid;
        g->planner_gen = g->d.planner->generation;
    }
    if (rc) release(g);
    ++g->captures;
    return rc;
}

}  // namespace

extern "C" {

int dcp_layer_graph_create(dcp_ctx* ctx, const dcp_layer_graph_desc* d, dcp_layer_graph** out) {
    DCP_REQUIRE(ctx && d && out && d->xchg && d->view && d->attn, DCP_E_INVALID_ARG, "NULL argument");
    DCP_REQUIRE(d->view->instance == d->xchg->cfg.self, DCP_E_INVALID_ARG, "view/instance mismatch");
    DCP_REQUIRE(d->xchg->committed, DCP_E_INVALID_ARG, "exchange not committed (dcp_xchg_commit)");
    if (d->moe) {
        DCP_REQUIRE(d->moe->committed, DCP_E_INVALID_ARG, "MoE exchange not committed (dcp_moe_commit)");
        DCP_REQUIRE(d->moe->cfg.self == d->view->instance && d->moe->cfg.world == d->view->world,
                    DCP_E_INVALID_ARG, "MoE exchange belongs to another instance / world");
        DCP_REQUIRE(d->y_region && d->moe_out, DCP_E_INVALID_ARG, "y_region / moe_out are required with MoE");
        DCP_REQUIRE(d->moe->cfg.m_max >= d->view->m_rows, DCP_E_SHAPE_OVERFLOW, "M %d > MoE m_max %d",
                    d->view->m_rows, d->moe->cfg.m_max);
    }
    auto* g = new dcp_layer_graph();
    g->ctx = ctx;
    g->d = *d;
    g->view = *d->view;
    g->attn = *d->attn;
    g->d.view = &g->view;
    g->d.attn = &g->attn;
    for (int m = 8;; m *= 2) {  // ShapeSpace M-hat ladder (routing.cpp:89-99), closed at m_max
        const int mh = m < d->xchg->cfg.m_max ? m : d->xchg->cfg.m_max;
        g->m_hat.push_back(mh);
        if (mh == d->xchg->cfg.m_max) break;
    }
    const int rc = capture_all(g);
    if (rc) {
        delete g;
        return rc;
    }
    *out = g;
    return DCP_OK;
}

int dcp_layer_graph_launch(dcp_layer_graph* g, int32_t m_rows, void* stream) {
    DCP_NVTX("layer graph replay");
    DCP_REQUIRE(g, DCP_E_INVALID_ARG, "NULL graph");
    DCP_REQUIRE(m_rows >= 0 && m_rows <= g->d.xchg->cfg.m_max, DCP_E_SHAPE_OVERFLOW, "M %d > m_max %d", m_rows,
                g->d.xchg->cfg.m_max);
    DCP_REQUIRE(!g->d.moe || m_rows <= g->d.moe->cfg.m_max, DCP_E_SHAPE_OVERFLOW, "M %d > MoE m_max %d", m_rows,
                g->d.moe->cfg.m_max);
    if (g->d.planner && g->d.planner->generation != g->planner_gen) {
        // the planner's page arena moved (compaction): the captured K7 holds stale pointers
        if (int rc = capture_all(g)) return rc;
    }
    size_t i = 0;
    while (g->m_hat[i] < m_rows) ++i;
    const int par = g->d.moe ? static_cast<int>((g->d.moe->host_epoch + 1) & 1) : 0;
    DCP_CUDA_TRY(cudaGraphLaunch(g->exec[par * g->m_hat.size() + i], static_cast<cudaStream_t>(stream)));
    if (g->d.moe) {  // the replayed step's host mirror (what dcp_moe_begin_step / dispatch / receive do)
        ++g->d.moe->host_epoch;
        g->d.moe->received = true;
        g->d.moe->m_count_dev = g->view.m_count_all + g->view.instance;
    }
    if (g->d.planner) g->d.planner->routing_valid = true;
    return DCP_OK;
}

int dcp_layer_graph_info(const dcp_layer_graph* g, int32_t* buckets, int32_t* captures) {
    DCP_REQUIRE(g, DCP_E_INVALID_ARG, "NULL graph");
    if (buckets) *buckets = static_cast<int32_t>(g->m_hat.size());
    if (captures) *captures = g->captures;
    return static_cast<int>(g->exec.size());
}

int dcp_layer_graph_destroy(dcp_layer_graph* g) {
    if (!g) return DCP_OK;
    release(g);
    delete g;
    return DCP_OK;
}

}  // extern "C"
