// SPDX-License-Identifier: Apache-2.0
// C ABI: device planner (K6) + routing lowering (K7).  See dcp_capi.h.
#include <algorithm>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include <cuda_bf16.h>

#include "capi_common.cuh"
#include "planner.cuh"
#include "routing.cuh"
#include "planner_internal.cuh"

using namespace dcp;

namespace {

__global__ void init_stacks_kernel(int32_t* stack, int W, int64_t cap) {
    const int64_t total = (int64_t)W * cap;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t f = i % cap;
        stack[i] = static_cast<int32_t>(cap - 1 - f);  // make_cluster: ascending hand-out
    }
}

// K8: one warp per M row; 16-byte stores of the new K and V rows of every
// kv-head into the (frame, slot) of the request's last page.
__global__ void kv_append_kernel(PlannerState st, const int32_t* m_slot, const int32_t* m_count,
                                 const __nv_bfloat16* kv_new, __nv_bfloat16* const* pools, int hkv, int d) {
    const int M = *m_count;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nwarps = (gridDim.x * blockDim.x) >> 5;
    for (int r = warp; r < M; r += nwarps) {
        const int sl = m_slot[r];
        if (st.last_append[sl] < 0) continue;  // growth stall: the token was not added
        const int c = st.page_cnt[sl];
        const int64_t last = st.page_off[sl] + c - 1;
        const int tgt = st.pg_inst[last];
        const int64_t frame = st.pg_frame[last];
        const int64_t slot = st.trailing_fill[sl] - 1;
        const int vec = d / 8;
        for (int i = lane; i < 2 * hkv * vec; i += 32) {
            const int kvh = i / vec, v = i % vec;  // kvh = kv * hkv + head
            const uint4* src = reinterpret_cast<const uint4*>(kv_new + ((size_t)r * 2 * hkv + kvh) * d) + v;
            uint4* dst = reinterpret_cast<uint4*>(pools[tgt] + (((frame * 2 * hkv) + kvh) * st.page + slot) * d) + v;
            *dst = *src;
        }
    }
}

// KV migration (MIGRATE / TRANSFER): request blockIdx.y's prefill K and V,
// contiguous [len][hkv][row] (row = d * elem bytes), go into the frames its placement holds.
// Logical page j holds the request's tokens [sum_{i<j} fill_i, + fill_j) — allocate lays the
// pages out member by member in kv_binding order (page_table.cpp:28-44) and append_token only
// extends the list — so each CTA sums the fills before its page range, then walks its pages.
// Every (part, head, token) row is 16-byte vectors: consecutive threads take consecutive
// vectors of a row, so source reads and frame writes (local or over NVLink) are coalesced.
__global__ void __launch_bounds__(256) kv_migrate_kernel(PlannerState st, const int32_t* slots,
                                                         const char* const* src_k, const char* const* src_v,
                                                         char* const* pools, int hkv, int row_bytes) {
    const int sl = slots[blockIdx.y];
    const int64_t off = st.page_off[sl];
    const int cnt = st.page_cnt[sl];
    const int p0 = static_cast<int>((int64_t)blockIdx.x * cnt / gridDim.x);
    const int p1 = static_cast<int>((int64_t)(blockIdx.x + 1) * cnt / gridDim.x);
    if (p0 >= p1) return;
    __shared__ int64_t s_part[8];
    int64_t before = 0;
    for (int j = threadIdx.x; j < p0; j += blockDim.x) before += st.pg_fill[off + j];
    for (int o = 16; o; o >>= 1) before += __shfl_xor_sync(0xffffffffu, before, o);
    if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = before;
    __syncthreads();
    int64_t tok0 = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tok0 += s_part[w];
    const int vec = row_bytes / 16;
    const char* k = src_k[blockIdx.y];
    const char* v = src_v[blockIdx.y];
    const int64_t page = st.page;
    for (int j = p0; j < p1; ++j) {
        const int inst = st.pg_inst[off + j];
        const int64_t frame = st.pg_frame[off + j];
        const int fill = st.pg_fill[off + j];
        char* fb = pools[inst] + frame * 2 * hkv * page * row_bytes;
        const int per_part = hkv * fill * vec;
        for (int i = threadIdx.x; i < 2 * per_part; i += blockDim.x) {
            const int part = i / per_part, rem = i % per_part;
            const int h = rem / (fill * vec), t = (rem / vec) % fill, x = rem % vec;
            const uint4* s = reinterpret_cast<const uint4*>((part ? v : k) + ((tok0 + t) * hkv + h) * row_bytes) + x;
            uint4* dd = reinterpret_cast<uint4*>(fb + ((part * hkv + h) * page + t) * row_bytes) + x;
            *dd = __ldg(s);
        }
        tok0 += fill;
    }
}

__global__ void enqueue_kernel(PlannerState st, const int32_t* slots, const int64_t* ids,
                               const int64_t* lens, int n) {
    const int base = *st.nwait;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int sl = slots[i];
        st.id[sl] = ids[i];
        st.seq_len[sl] = lens[i];
        st.generated[sl] = 0;
        st.state[sl] = ST_WAITING;
        st.k[sl] = 0;
        st.moe[sl] = -1;
        st.page_cnt[sl] = 0;
        st.page_cap[sl] = 0;
        st.trailing_fill[sl] = 0;
        st.last_append[sl] = -1;
        st.waiting[base + i] = sl;
    }
    __syncthreads();
    if (threadIdx.x == 0) *st.nwait = base + n;
}

template <class T>
int dalloc(T** p, size_t n, std::vector<void*>& owned) {
    void* q = nullptr;
    DCP_CUDA_TRY(cudaMalloc(&q, std::max<size_t>(n, 1) * sizeof(T)));
    DCP_CUDA_TRY(cudaMemset(q, 0, std::max<size_t>(n, 1) * sizeof(T)));
    owned.push_back(q);
    *p = static_cast<T*>(q);
    return DCP_OK;
}

int64_t pages_for_h(int64_t t, int64_t p) { return (t + p - 1) / p; }

}  // namespace


namespace {

int sync_arena_top(dcp_planner* pl) {
    DCP_CUDA_TRY(cudaStreamSynchronize(pl->stream));
    DCP_CUDA_TRY(cudaMemcpy(&pl->arena_top_host, pl->st.arena_top, sizeof(int64_t), cudaMemcpyDeviceToHost));
    return DCP_OK;
}

int compact_arena(dcp_planner* pl) {
    PlannerState& st = pl->st;
    planner_compact_offsets<<<1, 1024, 0, pl->stream>>>(st, pl->d_new_off);
    planner_compact_copy<<<st.max_slots, 128, 0, pl->stream>>>(st, pl->d_new_off, pl->arena2_inst,
                                                               pl->arena2_frame, pl->arena2_fill);
    DCP_CUDA_TRY(cudaGetLastError());
    std::swap(st.pg_inst, pl->arena2_inst);
    std::swap(st.pg_frame, pl->arena2_frame);
    std::swap(st.pg_fill, pl->arena2_fill);
    ++pl->generation;  // captured graphs holding the old arena pointers must be re-captured
    return sync_arena_top(pl);
}

void set_stream(dcp_planner* pl, void* s) { pl->stream = static_cast<cudaStream_t>(s); }

}  // namespace

namespace dcp {
int planner_sync_arena_top(dcp_planner* pl) { return sync_arena_top(pl); }
int planner_compact(dcp_planner* pl) { return compact_arena(pl); }
}  // namespace dcp

extern "C" {

int dcp_planner_create(dcp_ctx* ctx, const dcp_planner_config* c, dcp_planner** out) {
    DCP_REQUIRE(ctx && c && out, DCP_E_INVALID_ARG, "NULL argument");
    const int W = c->nodes * c->instances_per_node;
    DCP_REQUIRE(c->nodes >= 1 && c->instances_per_node >= 1, DCP_E_CONFIG, "empty topology");
    DCP_REQUIRE(W <= PL_MAXW, DCP_E_UNSUPPORTED, "world size %d > %d", W, PL_MAXW);
    DCP_REQUIRE(c->instances_per_node <= PL_MAXK, DCP_E_UNSUPPORTED, "instances_per_node %d > %d",
                c->instances_per_node, PL_MAXK);
    DCP_REQUIRE(c->page_size >= 1, DCP_E_CONFIG, "page_size < 1");
    // per-page fills are stored in 8 bits (pg_fill, routing page_fill)
    DCP_REQUIRE(c->page_size <= 255, DCP_E_UNSUPPORTED, "page_size %lld > 255", (long long)c->page_size);
    DCP_REQUIRE(c->capacity_pages >= 0 && c->capacity_pages < (1LL << 31), DCP_E_UNSUPPORTED,
                "capacity_pages out of range");
    DCP_REQUIRE(c->max_requests >= 1, DCP_E_INVALID_ARG, "max_requests < 1");
    // B_s sums stay below 2^22, which the planner's packed warp argmin relies on (planner.cuh)
    DCP_REQUIRE(c->max_requests <= (1 << 22) / PL_MAXW, DCP_E_INVALID_ARG, "max_requests %d > %d", c->max_requests,
                (1 << 22) / PL_MAXW);
    DCP_REQUIRE(c->policy >= 0 && c->policy <= 3, DCP_E_CONFIG, "unknown policy %d", c->policy);
    DCP_REQUIRE(c->n_bucket >= 0 && c->n_bucket <= 16, DCP_E_UNSUPPORTED, "n_bucket > 16");
    DCP_CUDA_TRY(cudaSetDevice(ctx->device));

    auto* pl = new dcp_planner();
    pl->ctx = ctx;
    pl->cfg = *c;
    PlannerState& st = pl->st;
    st.nodes = c->nodes;
    st.ipn = c->instances_per_node;
    st.W = W;
    st.kind = c->policy;
    st.udeg = c->uniform_degree;
    st.hol_strict = c->hol_strict;
    st.page = c->page_size;
    st.capacity = c->capacity_pages;
    st.max_slots = c->max_requests;
    st.reserve_pages = std::max<int64_t>(c->reserve_pages, 1);
    if (c->n_bucket == 0) {  // BucketFn::default_table (scheduler.cpp:28-33)
        const int64_t L[4] = {32768, 131072, 393216, INT64_MAX};
        const int32_t D[4] = {1, 2, 4, 8};
        st.nbucket = 4;
        for (int i = 0; i < 4; ++i) { st.bucket_len[i] = L[i]; st.bucket_deg[i] = D[i]; }
    } else {
        st.nbucket = c->n_bucket;
        for (int i = 0; i < c->n_bucket; ++i) {
            st.bucket_len[i] = c->bucket_len[i];
            st.bucket_deg[i] = c->bucket_deg[i];
        }
    }
    // SchedulerPolicy::validate (scheduler.cpp:35-41)
    if (st.kind == DCP_POLICY_DCP) {
        int64_t pl_ = 0;
        int pd = 0;
        bool bad = st.nbucket == 0;
        for (int i = 0; i < st.nbucket; ++i) {
            if (st.bucket_len[i] <= pl_ || st.bucket_deg[i] < pd || st.bucket_deg[i] < 1) bad = true;
            pl_ = st.bucket_len[i];
            pd = st.bucket_deg[i];
        }
        if (bad) {
            delete pl;
            set_error("bucket lengths must strictly increase and degrees be >=1, non-decreasing");
            return DCP_E_CONFIG;
        }
    }
    if (st.kind == DCP_POLICY_UNIFORM_CP) {
        if (st.udeg < 1 || st.ipn % st.udeg != 0) {
            delete pl;
            set_error("UniformCP degree must divide instances_per_node");
            return DCP_E_CONFIG;
        }
        st.n_groups = (st.ipn / st.udeg) * st.nodes;
    } else {
        st.n_groups = 1;
    }
    const size_t S = c->max_requests;
    int sort_cap = 1;
    while (sort_cap < (int)S) sort_cap <<= 1;
    st.sort_cap = sort_cap;
    st.arena_cap = 2 * (int64_t)W * c->capacity_pages + (int64_t)S * (PL_MAXK + st.reserve_pages) + 1024;

    auto& o = pl->owned;
    int rc = 0;
    rc |= dalloc(&st.kv_load, W, o);
    rc |= dalloc(&st.moe_batch, W, o);
    rc |= dalloc(&st.shard_count, W, o);
    rc |= dalloc(&st.nfree, W, o);
    rc |= dalloc(&st.stack, (size_t)W * c->capacity_pages, o);
    rc |= dalloc(&st.ucp_rr, st.n_groups, o);
    rc |= dalloc(&st.id, S, o);
    rc |= dalloc(&st.seq_len, S, o);
    rc |= dalloc(&st.generated, S, o);
    rc |= dalloc(&st.state, S, o);
    rc |= dalloc(&st.k, S, o);
    rc |= dalloc(&st.moe, S, o);
    rc |= dalloc(&st.kv, S * PL_MAXK, o);
    rc |= dalloc(&st.split, S * PL_MAXK, o);
    rc |= dalloc(&st.page_off, S, o);
    rc |= dalloc(&st.page_cnt, S, o);
    rc |= dalloc(&st.page_cap, S, o);
    rc |= dalloc(&st.trailing_fill, S, o);
    rc |= dalloc(&st.shard_tokens, S * W, o);
    rc |= dalloc(&st.last_append, S, o);
    rc |= dalloc(&st.pg_inst, st.arena_cap, o);
    rc |= dalloc(&st.pg_frame, st.arena_cap, o);
    rc |= dalloc(&st.pg_fill, st.arena_cap, o);
    rc |= dalloc(&pl->arena2_inst, st.arena_cap, o);
    rc |= dalloc(&pl->arena2_frame, st.arena_cap, o);
    rc |= dalloc(&pl->arena2_fill, st.arena_cap, o);
    rc |= dalloc(&pl->d_new_off, S, o);
    rc |= dalloc(&st.arena_top, 1, o);
    rc |= dalloc(&st.waiting, S, o);
    rc |= dalloc(&st.nwait, 1, o);
    rc |= dalloc(&st.res_slots, 3 * S, o);
    rc |= dalloc(&st.res_counts, 4, o);
    rc |= dalloc(&st.res_hol, 1, o);
    rc |= dalloc(&st.recs, S, o);
    rc |= dalloc(&st.res_pages, 1, o);
    rc |= dalloc(&st.sk1, sort_cap, o);
    rc |= dalloc(&st.sk2, sort_cap, o);
    rc |= dalloc(&st.sval, sort_cap, o);
    rc |= dalloc(&pl->d_io_slots, S, o);
    rc |= dalloc(&pl->d_io_ids, S, o);
    rc |= dalloc(&pl->d_io_lens, S, o);
    rc |= dalloc(&pl->d_io_out, S, o);
    RoutingOut& ro = pl->ro;
    rc |= dalloc(&ro.n_count, W, o);
    rc |= dalloc(&ro.n_active, 1, o);
    rc |= dalloc(&ro.m_count, W, o);
    rc |= dalloc(&ro.n_id, (size_t)W * S, o);
    rc |= dalloc(&ro.n_slot, (size_t)W * S, o);
    rc |= dalloc(&ro.n_moe, (size_t)W * S, o);
    rc |= dalloc(&ro.q_route, (size_t)W * S * W, o);
    rc |= dalloc(&ro.m_id, (size_t)W * S, o);
    rc |= dalloc(&ro.m_slot, (size_t)W * S, o);
    rc |= dalloc(&ro.res_route, (size_t)W * S * W, o);
    rc |= dalloc(&ro.bucket, 2 * W, o);
    rc |= dalloc(&ro.cu_pages, (size_t)W * (S + 1), o);
    rc |= dalloc(&ro.shard_len, (size_t)W * S, o);
    rc |= dalloc(&ro.block_table, (size_t)W * std::max<int64_t>(c->capacity_pages, 1), o);
    rc |= dalloc(&ro.page_fill, (size_t)W * std::max<int64_t>(c->capacity_pages, 1), o);
    rc |= dalloc(&ro.status, 1, o);
    rc |= dalloc(&ro.slot_nrow, S * W, o);
    rc |= dalloc(&ro.slot_mrow, S, o);
    rc |= dalloc(&ro.n_mrow, (size_t)W * S, o);
    rc |= dalloc(&ro.m_nrow, (size_t)W * S * W, o);
    rc |= dalloc(&ro.m_k, (size_t)W * S, o);
    rc |= dalloc(&ro.m_kv, (size_t)W * S * PL_MAXK, o);
    if (rc) {
        dcp_planner_destroy(pl);
        return DCP_E_CUDA;
    }
    // make_cluster: every instance starts with `capacity` free frames, LIFO stack
    std::vector<int64_t> nf(W, c->capacity_pages);
    DCP_CUDA_TRY(cudaMemcpy(st.nfree, nf.data(), W * sizeof(int64_t), cudaMemcpyHostToDevice));
    {
        std::vector<int32_t> fs(S, ST_FREE);
        DCP_CUDA_TRY(cudaMemcpy(st.state, fs.data(), S * sizeof(int32_t), cudaMemcpyHostToDevice));
    }
    if (c->capacity_pages > 0) init_stacks_kernel<<<256, 256>>>(st.stack, W, c->capacity_pages);
    DCP_CUDA_TRY(cudaGetLastError());
    DCP_CUDA_TRY(cudaDeviceSynchronize());
    pl->id_of_slot.assign(S, -1);
    pl->queued_len.assign(S, 0);
    pl->is_active.assign(S, 0);
    for (int i = (int)S - 1; i >= 0; --i) pl->free_slots.push_back(i);
    *out = pl;
    return DCP_OK;
}

int dcp_planner_destroy(dcp_planner* pl) {
    if (!pl) return DCP_OK;
    for (void* p : pl->owned) cudaFree(p);
    delete pl;
    return DCP_OK;
}

int dcp_planner_last_launches(const dcp_planner* pl) { return pl ? pl->last_launches : 0; }

int dcp_planner_enqueue(dcp_planner* pl, const int64_t* ids, const int64_t* lens, int32_t n) {
    DCP_REQUIRE(pl && (n == 0 || (ids && lens)), DCP_E_INVALID_ARG, "NULL argument");
    if (n == 0) return DCP_OK;
    DCP_REQUIRE((size_t)n <= pl->free_slots.size(), DCP_E_INVALID_ARG,
                "request slots exhausted (max_requests=%d)", pl->cfg.max_requests);
    std::vector<int32_t> slots(n);
    for (int i = 0; i < n; ++i) {
        DCP_REQUIRE(!pl->slot_of.count(ids[i]), DCP_E_INVALID_ARG, "request id %lld already tracked",
                    (long long)ids[i]);
    }
    for (int i = 0; i < n; ++i) pl->retired.erase(ids[i]);
    for (int i = 0; i < n; ++i) {
        const int sl = pl->free_slots.back();
        pl->free_slots.pop_back();
        slots[i] = sl;
        pl->slot_of[ids[i]] = sl;
        pl->id_of_slot[sl] = ids[i];
        pl->queued_len[sl] = lens[i];
        pl->waiting_pages_bound +=
            pages_for_h(std::max<int64_t>(lens[i], 0), pl->cfg.page_size) + PL_MAXK + pl->st.reserve_pages;
    }
    pl->queued += n;
    DCP_CUDA_TRY(cudaMemcpyAsync(pl->d_io_slots, slots.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice, pl->stream));
    DCP_CUDA_TRY(cudaMemcpyAsync(pl->d_io_ids, ids, n * sizeof(int64_t), cudaMemcpyHostToDevice, pl->stream));
    DCP_CUDA_TRY(cudaMemcpyAsync(pl->d_io_lens, lens, n * sizeof(int64_t), cudaMemcpyHostToDevice, pl->stream));
    enqueue_kernel<<<1, 256, 0, pl->stream>>>(pl->st, pl->d_io_slots, pl->d_io_ids, pl->d_io_lens, n);
    DCP_CUDA_TRY(cudaGetLastError());
    DCP_CUDA_TRY(cudaStreamSynchronize(pl->stream));  // staging buffers are reused
    return DCP_OK;
}

int dcp_planner_step(dcp_planner* pl, void* stream) {
    DCP_NVTX("K6 planner step");
    DCP_REQUIRE(pl, DCP_E_INVALID_ARG, "NULL planner");
    set_stream(pl, stream);
    pl->last_launches = 0;
    if (pl->arena_top_host + pl->waiting_pages_bound > pl->st.arena_cap) {
        int rc = compact_arena(pl);
        if (rc) return rc;
        pl->last_launches += 2;
    }
    planner_step_kernel<<<1, PL_THREADS, 0, pl->stream>>>(pl->st);
    DCP_CUDA_TRY(cudaGetLastError());
    DCP_CUDA_TRY(launch_pdl(planner_pages_kernel, dim3(pl->ctx->num_sms * 2), dim3(256), 0, pl->stream, pl->st));
    pl->last_launches += 2;
    pl->routing_valid = false;
    // conservative bound until the result is read back
    pl->arena_top_host += pl->waiting_pages_bound;
    return DCP_OK;
}

int dcp_planner_step_result(dcp_planner* pl, int64_t* committed, int32_t* nc, int64_t* deferred,
                            int32_t* nd, int64_t* unsched, int32_t* nu, int64_t* hol) {
    DCP_REQUIRE(pl && nc && nd && nu && hol, DCP_E_INVALID_ARG, "NULL argument");
    DCP_CUDA_TRY(cudaStreamSynchronize(pl->stream));
    int32_t cnt[4];
    DCP_CUDA_TRY(cudaMemcpy(cnt, pl->st.res_counts, sizeof(cnt), cudaMemcpyDeviceToHost));
    DCP_CUDA_TRY(cudaMemcpy(hol, pl->st.res_hol, sizeof(int64_t), cudaMemcpyDeviceToHost));
    const size_t S = pl->cfg.max_requests;
    std::vector<int32_t> sl(3 * S);
    DCP_CUDA_TRY(cudaMemcpy(sl.data(), pl->st.res_slots, 3 * S * sizeof(int32_t), cudaMemcpyDeviceToHost));
    *nc = cnt[0];
    *nd = cnt[1];
    *nu = cnt[2];
    for (int i = 0; i < cnt[0]; ++i) {
        const int s = sl[i];
        if (committed) committed[i] = pl->id_of_slot[s];
        pl->is_active[s] = 1;
        pl->waiting_pages_bound -=
            pages_for_h(pl->queued_len[s], pl->cfg.page_size) + PL_MAXK + pl->st.reserve_pages;
        pl->queued -= 1;
    }
    for (int i = 0; i < cnt[1]; ++i)
        if (deferred) deferred[i] = pl->id_of_slot[sl[S + i]];
    for (int i = 0; i < cnt[2]; ++i) {
        const int s = sl[2 * S + i];
        const int64_t id = pl->id_of_slot[s];
        if (unsched) unsched[i] = id;
        // erased from the queue and never placed: release the slot
        pl->waiting_pages_bound -=
            pages_for_h(pl->queued_len[s], pl->cfg.page_size) + PL_MAXK + pl->st.reserve_pages;
        pl->queued -= 1;
        pl->slot_of.erase(id);
        pl->id_of_slot[s] = -1;
        pl->free_slots.push_back(s);
    }
    DCP_CUDA_TRY(cudaMemcpy(&pl->arena_top_host, pl->st.arena_top, sizeof(int64_t), cudaMemcpyDeviceToHost));
    if (cnt[3] == PL_E_FRAMES) {
        set_error("cannot allocate a zero-length request");
        return DCP_E_INSUFFICIENT_FRAMES;
    }
    if (cnt[3] != 0) {
        set_error("planner step status %d", cnt[3]);
        return DCP_E_CUDA;
    }
    return DCP_OK;
}

int dcp_planner_finish(dcp_planner* pl, const int64_t* ids, int32_t n, void* stream) {
    DCP_REQUIRE(pl && (n == 0 || ids), DCP_E_INVALID_ARG, "NULL argument");
    if (n == 0) return DCP_OK;
    set_stream(pl, stream);
    std::vector<int32_t> slots;
    std::vector<int32_t> st(n);
    for (int i = 0; i < n; ++i) {
        auto it = pl->slot_of.find(ids[i]);
        DCP_REQUIRE(it != pl->slot_of.end(), DCP_E_UNKNOWN_REQUEST,
                    "no page-table entries for request %lld", (long long)ids[i]);
        slots.push_back(it->second);
    }
    // only ACTIVE requests have page-table entries (UnknownRequest otherwise)
    for (int i = 0; i < n; ++i)
        DCP_REQUIRE(pl->is_active[slots[i]], DCP_E_UNKNOWN_REQUEST, "no page-table entries for request %lld",
                    (long long)ids[i]);
    for (int i = 0; i < n; ++i) {
        dcp_planner::Retired r{};
        DCP_CUDA_TRY(cudaMemcpy(&r.k, pl->st.k + slots[i], 4, cudaMemcpyDeviceToHost));
        DCP_CUDA_TRY(cudaMemcpy(&r.moe, pl->st.moe + slots[i], 4, cudaMemcpyDeviceToHost));
        DCP_CUDA_TRY(cudaMemcpy(r.kv, pl->st.kv + (size_t)slots[i] * PL_MAXK, r.k * 4, cudaMemcpyDeviceToHost));
        DCP_CUDA_TRY(cudaMemcpy(r.split, pl->st.split + (size_t)slots[i] * PL_MAXK, r.k * 8, cudaMemcpyDeviceToHost));
        pl->retired[ids[i]] = r;
    }
    DCP_CUDA_TRY(cudaMemcpyAsync(pl->d_io_slots, slots.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice, pl->stream));
    planner_release_kernel<<<1, PL_THREADS, 0, pl->stream>>>(pl->st, pl->d_io_slots, n);
    DCP_CUDA_TRY(cudaGetLastError());
    DCP_CUDA_TRY(cudaStreamSynchronize(pl->stream));
    for (int i = 0; i < n; ++i) {
        pl->slot_of.erase(ids[i]);
        pl->id_of_slot[slots[i]] = -1;
        pl->is_active[slots[i]] = 0;
        pl->free_slots.push_back(slots[i]);
    }
    pl->routing_valid = false;
    pl->last_launches = 1;
    return DCP_OK;
}

int dcp_planner_append_token(dcp_planner* pl, const int64_t* ids, int32_t n, int32_t* out_inst) {
    DCP_REQUIRE(pl && (n == 0 || (ids && out_inst)), DCP_E_INVALID_ARG, "NULL argument");
    std::vector<int32_t> slots(n);
    for (int i = 0; i < n; ++i) {
        auto it = pl->slot_of.find(ids[i]);
        DCP_REQUIRE(it != pl->slot_of.end(), DCP_E_UNKNOWN_REQUEST, "unknown request %lld",
                    (long long)ids[i]);
        DCP_REQUIRE(pl->is_active[it->second], DCP_E_UNKNOWN_REQUEST, "no page-table entries for request %lld",
                    (long long)ids[i]);
        slots[i] = it->second;
    }
    int done = 0;
    int guard = 0;
    // Batches without duplicate requests take the parallel kernel; it declines
    // (res_counts[2] = 1, nothing mutated) when a frame fallback could occur.
    bool unique = true;
    {
        std::vector<int32_t> sorted(slots);
        std::sort(sorted.begin(), sorted.end());
        unique = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
    }
    if (unique && n > 0) {
        DCP_CUDA_TRY(cudaMemcpyAsync(pl->d_io_slots, slots.data(), n * sizeof(int32_t), cudaMemcpyHostToDevice,
                                     pl->stream));
        planner_append_parallel_kernel<<<1, PL_APPEND_THREADS, 0, pl->stream>>>(pl->st, pl->d_io_slots, n,
                                                                               pl->d_io_out);
        DCP_CUDA_TRY(cudaGetLastError());
        int32_t cnt[4];
        DCP_CUDA_TRY(cudaMemcpyAsync(cnt, pl->st.res_counts, sizeof(cnt), cudaMemcpyDeviceToHost, pl->stream));
        DCP_CUDA_TRY(cudaStreamSynchronize(pl->stream));
        if (cnt[2] == 0) {
            DCP_CUDA_TRY(cudaMemcpy(out_inst, pl->d_io_out, n * sizeof(int32_t), cudaMemcpyDeviceToHost));
            done = n;
        }
    }
    while (done < n) {
        const int m = n - done;
        DCP_CUDA_TRY(cudaMemcpyAsync(pl->d_io_slots, slots.data() + done, m * sizeof(int32_t),
                                     cudaMemcpyHostToDevice, pl->stream));
        planner_append_kernel<<<1, 32, 0, pl->stream>>>(pl->st, pl->d_io_slots, m, pl->d_io_out);
        DCP_CUDA_TRY(cudaGetLastError());
        DCP_CUDA_TRY(cudaStreamSynchronize(pl->stream));
        int32_t cnt[4];
        DCP_CUDA_TRY(cudaMemcpy(cnt, pl->st.res_counts, sizeof(cnt), cudaMemcpyDeviceToHost));
        DCP_CUDA_TRY(cudaMemcpy(out_inst + done, pl->d_io_out, cnt[0] * sizeof(int32_t), cudaMemcpyDeviceToHost));
        done += cnt[0];
        if (cnt[3] == PL_E_ARENA) {
            DCP_REQUIRE(++guard < 4, DCP_E_CUDA, "page arena exhausted");
            int rc = compact_arena(pl);
            if (rc) return rc;
        }
    }
    DCP_CUDA_TRY(cudaMemcpy(&pl->arena_top_host, pl->st.arena_top, sizeof(int64_t), cudaMemcpyDeviceToHost));
    pl->routing_valid = false;
    return DCP_OK;
}

int dcp_planner_placement(dcp_planner* pl, int64_t id, int32_t* kv, int64_t* split, int32_t* moe,
                          int32_t* k) {
    DCP_REQUIRE(pl && kv && split && moe && k, DCP_E_INVALID_ARG, "NULL argument");
    auto it = pl->slot_of.find(id);
    if (it == pl->slot_of.end()) {
        auto rt = pl->retired.find(id);
        DCP_REQUIRE(rt != pl->retired.end(), DCP_E_UNKNOWN_REQUEST, "unknown request %lld", (long long)id);
        *k = rt->second.k;
        *moe = rt->second.moe;
        for (int m = 0; m < *k; ++m) {
            kv[m] = rt->second.kv[m];
            split[m] = rt->second.split[m];
        }
        return DCP_OK;
    }
    const int sl = it->second;
    DCP_CUDA_TRY(cudaStreamSynchronize(pl->stream));
    int32_t state = 0;
    DCP_CUDA_TRY(cudaMemcpy(&state, pl->st.state + sl, sizeof(int32_t), cudaMemcpyDeviceToHost));
    DCP_REQUIRE(state == ST_ACTIVE, DCP_E_UNKNOWN_REQUEST, "request %lld has no placement", (long long)id);
    DCP_CUDA_TRY(cudaMemcpy(k, pl->st.k + sl, sizeof(int32_t), cudaMemcpyDeviceToHost));
    DCP_CUDA_TRY(cudaMemcpy(moe, pl->st.moe + sl, sizeof(int32_t), cudaMemcpyDeviceToHost));
    DCP_CUDA_TRY(cudaMemcpy(kv, pl->st.kv + (size_t)sl * PL_MAXK, *k * sizeof(int32_t), cudaMemcpyDeviceToHost));
    DCP_CUDA_TRY(cudaMemcpy(split, pl->st.split + (size_t)sl * PL_MAXK, *k * sizeof(int64_t), cudaMemcpyDeviceToHost));
    return DCP_OK;
}

int dcp_planner_instances(dcp_planner* pl, int64_t* kv_load, int32_t* moe_batch, int32_t* shard_count,
                          int64_t* free_frames) {
    DCP_REQUIRE(pl, DCP_E_INVALID_ARG, "NULL planner");
    DCP_CUDA_TRY(cudaStreamSynchronize(pl->stream));
    const int W = pl->st.W;
    if (kv_load) DCP_CUDA_TRY(cudaMemcpy(kv_load, pl->st.kv_load, W * 8, cudaMemcpyDeviceToHost));
    if (moe_batch) DCP_CUDA_TRY(cudaMemcpy(moe_batch, pl->st.moe_batch, W * 4, cudaMemcpyDeviceToHost));
    if (shard_count) DCP_CUDA_TRY(cudaMemcpy(shard_count, pl->st.shard_count, W * 4, cudaMemcpyDeviceToHost));
    if (free_frames) DCP_CUDA_TRY(cudaMemcpy(free_frames, pl->st.nfree, W * 8, cudaMemcpyDeviceToHost));
    return W;
}

static int64_t emit(const std::string& s, char* buf, int64_t cap) {
    if (buf && cap > 0) {
        const int64_t n = std::min<int64_t>((int64_t)s.size(), cap - 1);
        std::memcpy(buf, s.data(), n);
        buf[n] = 0;
    }
    return (int64_t)s.size();
}

int64_t dcp_planner_dump_page_table(dcp_planner* pl, char* buf, int64_t cap) {
    if (!pl) return DCP_E_INVALID_ARG;
    if (cudaStreamSynchronize(pl->stream) != cudaSuccess) return DCP_E_CUDA;
    const size_t S = pl->cfg.max_requests;
    std::vector<int32_t> state(S), cnt(S);
    std::vector<int64_t> off(S), id(S);
    int64_t top = 0;
    cudaMemcpy(state.data(), pl->st.state, S * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(cnt.data(), pl->st.page_cnt, S * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(off.data(), pl->st.page_off, S * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(id.data(), pl->st.id, S * 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&top, pl->st.arena_top, 8, cudaMemcpyDeviceToHost);
    std::vector<int32_t> inst(top), frame(top);
    if (top) {
        cudaMemcpy(inst.data(), pl->st.pg_inst, top * 4, cudaMemcpyDeviceToHost);
        cudaMemcpy(frame.data(), pl->st.pg_frame, top * 4, cudaMemcpyDeviceToHost);
    }
    if (cudaGetLastError() != cudaSuccess) return DCP_E_CUDA;
    std::vector<std::pair<int64_t, int>> live;
    for (size_t s = 0; s < S; ++s)
        if (state[s] == ST_ACTIVE) live.push_back({id[s], (int)s});
    std::sort(live.begin(), live.end());
    std::string out = "request_id,logical_page,instance_id,frame_id\n";
    char line[96];
    for (auto& [rid, s] : live)
        for (int p = 0; p < cnt[s]; ++p) {
            std::snprintf(line, sizeof(line), "%lld,%d,%d,%d\n", (long long)rid, p, inst[off[s] + p],
                          frame[off[s] + p]);
            out += line;
        }
    return emit(out, buf, cap);
}

int dcp_planner_build_routing(dcp_planner* pl, void* stream) {
    DCP_NVTX("K7 routing tables");
    DCP_REQUIRE(pl, DCP_E_INVALID_ARG, "NULL planner");
    set_stream(pl, stream);
    DCP_CUDA_TRY(launch_routing_rows(pl->st, pl->ro, pl->stream));
    const dim3 wide(pl->st.W, RT_SPLIT);
    DCP_CUDA_TRY(launch_pdl(routing_count_kernel, wide, dim3(256), 0, pl->stream, pl->st, pl->ro));
    DCP_CUDA_TRY(launch_pdl(routing_scan_kernel, dim3(pl->st.W), dim3(1024), 0, pl->stream, pl->st, pl->ro));
    DCP_CUDA_TRY(launch_pdl(routing_scatter_kernel, wide, dim3(256), 0, pl->stream, pl->st, pl->ro));
    pl->last_launches = ROWS_SMEM_MAX >= pl->st.max_slots ? 7 : 4;
    pl->routing_valid = true;
    return DCP_OK;
}

int64_t dcp_planner_dump_routing(dcp_planner* pl, char* buf, int64_t cap) {
    if (!pl) return DCP_E_INVALID_ARG;
    if (!pl->routing_valid) {
        int rc = dcp_planner_build_routing(pl, pl->stream);
        if (rc) return rc;
    }
    if (cudaStreamSynchronize(pl->stream) != cudaSuccess) return DCP_E_CUDA;
    int32_t status = 0;
    cudaMemcpy(&status, pl->ro.status, 4, cudaMemcpyDeviceToHost);
    if (status == -4) {
        set_error("moe_binding outside kv_binding");
        return DCP_E_INCONSISTENT;
    }
    const int W = pl->st.W;
    const size_t S = pl->cfg.max_requests;
    std::vector<int32_t> nc(W), mc(W);
    cudaMemcpy(nc.data(), pl->ro.n_count, W * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(mc.data(), pl->ro.m_count, W * 4, cudaMemcpyDeviceToHost);
    std::string out = "instance,table,row,request_id,columns\n";
    std::vector<int64_t> ids;
    std::vector<uint8_t> bits;
    char line[128];
    for (int s = 0; s < W; ++s) {
        for (int t = 0; t < 2; ++t) {
            const int rows = t == 0 ? nc[s] : mc[s];
            ids.resize(rows);
            bits.resize((size_t)rows * W);
            if (rows) {
                cudaMemcpy(ids.data(), (t == 0 ? pl->ro.n_id : pl->ro.m_id) + (size_t)s * S, rows * 8,
                           cudaMemcpyDeviceToHost);
                cudaMemcpy(bits.data(), (t == 0 ? pl->ro.q_route : pl->ro.res_route) + (size_t)s * S * W,
                           (size_t)rows * W, cudaMemcpyDeviceToHost);
            }
            for (int r = 0; r < rows; ++r) {
                std::snprintf(line, sizeof(line), "%d,%s,%d,%lld,", s, t == 0 ? "q_route" : "res_route", r,
                              (long long)ids[r]);
                out += line;
                for (int c = 0; c < W; ++c) out += bits[(size_t)r * W + c] ? '1' : '0';
                out += '\n';
            }
        }
    }
    if (cudaGetLastError() != cudaSuccess) return DCP_E_CUDA;
    return emit(out, buf, cap);
}

int dcp_kv_append(dcp_planner* pl, int32_t s, const void* kv_new, void* const* pools, int32_t hkv, int32_t d,
                  void* stream) {
    DCP_REQUIRE(pl && pools, DCP_E_INVALID_ARG, "NULL argument");
    DCP_REQUIRE(s >= 0 && s < pl->st.W, DCP_E_INVALID_ARG, "instance %d out of range", s);
    DCP_REQUIRE(pl->routing_valid, DCP_E_INVALID_ARG, "call dcp_planner_build_routing after append_token");
    DCP_REQUIRE(d % 8 == 0 && hkv >= 1, DCP_E_UNSUPPORTED, "head_dim %d", d);
    if (!pl->d_pools) {
        void* q = nullptr;
        DCP_CUDA_TRY(cudaMalloc(&q, PL_MAXW * sizeof(void*)));
        pl->owned.push_back(q);
        pl->d_pools = static_cast<__nv_bfloat16**>(q);
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    DCP_CUDA_TRY(cudaMemcpyAsync(pl->d_pools, pools, pl->st.W * sizeof(void*), cudaMemcpyHostToDevice, st));
    const size_t S = pl->cfg.max_requests;
    kv_append_kernel<<<64, 256, 0, st>>>(pl->st, pl->ro.m_slot + (size_t)s * S, pl->ro.m_count + s,
                                         static_cast<const __nv_bfloat16*>(kv_new), pl->d_pools, hkv, d);
    DCP_CUDA_TRY(cudaGetLastError());
    DCP_CUDA_TRY(cudaStreamSynchronize(st));  // the staged pool table is reused
    return DCP_OK;
}

int dcp_kv_migrate(dcp_planner* pl, const int64_t* ids, int32_t n, const void* const* src_k,
                   const void* const* src_v, void* const* pools, int32_t hkv, int32_t head_dim, int32_t elem_bytes,
                   void* stream) {
    DCP_NVTX("KV migrate");
    DCP_REQUIRE(pl && (n == 0 || (ids && src_k && src_v && pools)), DCP_E_INVALID_ARG, "NULL argument");
    DCP_REQUIRE(n >= 0 && n <= 65535, DCP_E_INVALID_ARG, "n %d", n);
    DCP_REQUIRE(hkv >= 1 && head_dim >= 1 && (elem_bytes == 2 || elem_bytes == 4), DCP_E_UNSUPPORTED,
                "elem_bytes %d", elem_bytes);
    const int row_bytes = head_dim * elem_bytes;
    DCP_REQUIRE(row_bytes % 16 == 0, DCP_E_UNSUPPORTED, "head_dim x elem_bytes must be a multiple of 16");
    if (n == 0) return DCP_OK;
    const int W = pl->st.W;
    std::vector<int32_t> slots(n);
    for (int i = 0; i < n; ++i) {
        auto it = pl->slot_of.find(ids[i]);
        DCP_REQUIRE(it != pl->slot_of.end(), DCP_E_UNKNOWN_REQUEST, "unknown request %lld", (long long)ids[i]);
        DCP_REQUIRE(pl->is_active[it->second], DCP_E_INVALID_ARG, "request %lld holds no pages (not admitted)",
                    (long long)ids[i]);
        DCP_REQUIRE(src_k[i] && src_v[i], DCP_E_INVALID_ARG, "NULL source of request %lld", (long long)ids[i]);
        DCP_REQUIRE((reinterpret_cast<uintptr_t>(src_k[i]) | reinterpret_cast<uintptr_t>(src_v[i])) % 16 == 0,
                    DCP_E_INVALID_ARG, "sources must be 16-byte aligned");
        slots[i] = it->second;
    }
    for (int s = 0; s < W; ++s) DCP_REQUIRE(pools[s], DCP_E_INVALID_ARG, "pool of instance %d is NULL", s);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // one staging block: slots | src_k | src_v | pools
    const size_t bytes = n * 4 + 8 + 2 * (size_t)n * 8 + (size_t)W * 8;
    std::vector<char> h(bytes);
    std::memcpy(h.data(), slots.data(), n * 4);
    const size_t ok = (n * 4 + 7) & ~size_t(7);
    std::memcpy(h.data() + ok, src_k, n * 8);
    std::memcpy(h.data() + ok + n * 8, src_v, n * 8);
    std::memcpy(h.data() + ok + 2 * n * 8, pools, W * 8);
    char* d = nullptr;
    DCP_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&d), bytes, st));
    DCP_CUDA_TRY(cudaMemcpyAsync(d, h.data(), bytes, cudaMemcpyHostToDevice, st));
    kv_migrate_kernel<<<dim3(64, n), 256, 0, st>>>(
        pl->st, reinterpret_cast<const int32_t*>(d), reinterpret_cast<const char* const*>(d + ok),
        reinterpret_cast<const char* const*>(d + ok + n * 8), reinterpret_cast<char* const*>(d + ok + 2 * n * 8),
        hkv, row_bytes);
    DCP_CUDA_TRY(cudaGetLastError());
    DCP_CUDA_TRY(cudaFreeAsync(d, st));  // h was staged by the pageable copy before it returned
    return DCP_OK;
}

int dcp_planner_instance_view(dcp_planner* pl, int32_t s, dcp_instance_view* v) {
    DCP_REQUIRE(pl && v, DCP_E_INVALID_ARG, "NULL argument");
    DCP_REQUIRE(s >= 0 && s < pl->st.W, DCP_E_INVALID_ARG, "instance %d out of range", s);
    DCP_REQUIRE(pl->routing_valid, DCP_E_INVALID_ARG, "call dcp_planner_build_routing first");
    DCP_CUDA_TRY(cudaStreamSynchronize(pl->stream));
    const size_t S = pl->cfg.max_requests;
    const int W = pl->st.W;
    int32_t b[2];
    DCP_CUDA_TRY(cudaMemcpy(&v->n_rows, pl->ro.n_count + s, 4, cudaMemcpyDeviceToHost));
    DCP_CUDA_TRY(cudaMemcpy(&v->m_rows, pl->ro.m_count + s, 4, cudaMemcpyDeviceToHost));
    DCP_CUDA_TRY(cudaMemcpy(b, pl->ro.bucket + 2 * s, 8, cudaMemcpyDeviceToHost));
    v->bucket_m = b[0];
    v->bucket_n = b[1];
    v->n_ids = pl->ro.n_id + (size_t)s * S;
    v->n_moe = pl->ro.n_moe + (size_t)s * S;
    v->q_route = pl->ro.q_route + (size_t)s * S * W;
    v->m_ids = pl->ro.m_id + (size_t)s * S;
    v->res_route = pl->ro.res_route + (size_t)s * S * W;
    v->cu_pages = pl->ro.cu_pages + (size_t)s * (S + 1);
    v->shard_len = pl->ro.shard_len + (size_t)s * S;
    v->block_table = pl->ro.block_table + (size_t)s * pl->st.capacity;
    v->page_fill = pl->ro.page_fill + (size_t)s * pl->st.capacity;
    v->n_mrow = pl->ro.n_mrow + (size_t)s * S;
    v->m_nrow = pl->ro.m_nrow + (size_t)s * S * W;
    v->m_k = pl->ro.m_k + (size_t)s * S;
    v->m_kv = pl->ro.m_kv + (size_t)s * S * PL_MAXK;
    v->m_count_all = pl->ro.m_count;
    v->n_count_dev = pl->ro.n_count + s;
    v->total_pages_dev = pl->ro.cu_pages + (size_t)s * (S + 1) + S;
    v->world = W;
    v->instance = s;
    return DCP_OK;
}

}  // extern "C"
