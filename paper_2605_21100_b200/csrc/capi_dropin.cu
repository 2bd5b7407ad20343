// SPDX-License-Identifier: Apache-2.0
// C ABI entry points that back the dcpsim C++ drop-in (include/dcpsim/):
// policy/queue synchronisation, explicit-placement allocation, standalone
// rebalance / water_fill / binding-config / routing-table expansion, and the
// fp32/fp64 contiguous attention math.  See dcp_capi.h.
#include <algorithm>
#include <cstring>
#include <vector>

#include "attn_contig.cuh"
#include "planner_internal.cuh"

using namespace dcp;

namespace {

__global__ void set_queue_kernel(PlannerState st, const int32_t* slots, const int64_t* ids,
                                 const int64_t* lens, const int32_t* is_new, int n,
                                 const int32_t* drop, int ndrop) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const int sl = slots[i];
        if (is_new[i]) {
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
        }
        st.waiting[i] = sl;
    }
    for (int j = threadIdx.x; j < ndrop; j += blockDim.x) st.state[drop[j]] = ST_FREE;
    __syncthreads();
    if (threadIdx.x == 0) *st.nwait = n;
}

__global__ void load_instances_kernel(PlannerState st, const int64_t* kv, const int32_t* b,
                                      const int32_t* sc, const int64_t* nf, const int32_t* stacks) {
    const int W = st.W;
    if (blockIdx.x == 0 && threadIdx.x < W) {
        st.kv_load[threadIdx.x] = kv[threadIdx.x];
        st.moe_batch[threadIdx.x] = b[threadIdx.x];
        st.shard_count[threadIdx.x] = sc[threadIdx.x];
        st.nfree[threadIdx.x] = nf[threadIdx.x];
    }
    const int64_t total = (int64_t)W * st.capacity;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x)
        st.stack[i] = stacks[i];
}

__global__ void route_expand_kernel(int W, int n, const int32_t* shard_moe, int m, const uint32_t* res_mask,
                                    uint8_t* q, uint8_t* res) {
    const int64_t tq = (int64_t)n * W, tr = (int64_t)m * W;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tq + tr;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (i < tq) {
            const int r = (int)(i / W), c = (int)(i % W);
            q[i] = c == shard_moe[r] ? 1 : 0;
        } else {
            const int64_t j = i - tq;
            const int r = (int)(j / W), c = (int)(j % W);
            res[j] = (res_mask[r] >> c) & 1u;
        }
    }
}

template <class T>
int dalloc_tmp(T** p, size_t n, std::vector<void*>& owned) {
    void* q = nullptr;
    DCP_CUDA_TRY(cudaMalloc(&q, std::max<size_t>(n, 1) * sizeof(T)));
    DCP_CUDA_TRY(cudaMemset(q, 0, std::max<size_t>(n, 1) * sizeof(T)));
    owned.push_back(q);
    *p = static_cast<T*>(q);
    return DCP_OK;
}

struct TmpFree {
    std::vector<void*> v;
    ~TmpFree() {
        for (void* p : v) cudaFree(p);
    }
};

int planner_states(dcp_planner* pl, std::vector<int32_t>& state) {
    const size_t S = pl->cfg.max_requests;
    state.resize(S);
    DCP_CUDA_TRY(cudaStreamSynchronize(pl->stream));
    DCP_CUDA_TRY(cudaMemcpy(state.data(), pl->st.state, S * 4, cudaMemcpyDeviceToHost));
    return DCP_OK;
}

}  // namespace

extern "C" {

int dcp_planner_set_policy(dcp_planner* pl, int32_t policy, int32_t n_bucket, const int64_t* bl,
                           const int32_t* bd, int32_t udeg, int32_t hol_strict) {
    DCP_REQUIRE(pl, DCP_E_INVALID_ARG, "NULL planner");
    DCP_REQUIRE(policy >= 0 && policy <= 3, DCP_E_CONFIG, "unknown policy %d", policy);
    DCP_REQUIRE(n_bucket >= 0 && n_bucket <= 16, DCP_E_UNSUPPORTED, "n_bucket > 16");
    PlannerState& st = pl->st;
    int64_t L[16];
    int32_t D[16];
    int nb = n_bucket;
    if (nb == 0) {
        const int64_t dl[4] = {32768, 131072, 393216, INT64_MAX};
        const int32_t dd[4] = {1, 2, 4, 8};
        nb = 4;
        for (int i = 0; i < 4; ++i) { L[i] = dl[i]; D[i] = dd[i]; }
    } else {
        for (int i = 0; i < nb; ++i) { L[i] = bl[i]; D[i] = bd[i]; }
    }
    if (policy == DCP_POLICY_DCP) {  // BucketFn::validate (scheduler.cpp:16-26)
        int64_t pl_ = 0;
        int pd = 0;
        for (int i = 0; i < nb; ++i) {
            DCP_REQUIRE(L[i] > pl_, DCP_E_CONFIG, "bucket lengths must strictly increase");
            DCP_REQUIRE(D[i] >= pd && D[i] >= 1, DCP_E_CONFIG, "bucket degrees must be >=1 and non-decreasing");
            pl_ = L[i];
            pd = D[i];
        }
    }
    int n_groups = 1;
    if (policy == DCP_POLICY_UNIFORM_CP) {
        DCP_REQUIRE(udeg >= 1 && st.ipn % udeg == 0, DCP_E_CONFIG,
                    "UniformCP degree must divide instances_per_node");
        n_groups = (st.ipn / udeg) * st.nodes;
    }
    if (policy == DCP_POLICY_UNIFORM_CP && (n_groups != st.n_groups || udeg != st.udeg)) {
        // the round-robin vector is re-assigned when its size changes
        DCP_CUDA_TRY(cudaFree(st.ucp_rr));
        auto it = std::find(pl->owned.begin(), pl->owned.end(), static_cast<void*>(st.ucp_rr));
        if (it != pl->owned.end()) pl->owned.erase(it);
        void* q = nullptr;
        DCP_CUDA_TRY(cudaMalloc(&q, n_groups * sizeof(int32_t)));
        DCP_CUDA_TRY(cudaMemset(q, 0, n_groups * sizeof(int32_t)));
        pl->owned.push_back(q);
        st.ucp_rr = static_cast<int32_t*>(q);
    }
    st.kind = policy;
    st.nbucket = nb;
    for (int i = 0; i < nb; ++i) {
        st.bucket_len[i] = L[i];
        st.bucket_deg[i] = D[i];
    }
    st.udeg = udeg;
    st.n_groups = n_groups;
    st.hol_strict = hol_strict;
    return DCP_OK;
}

int dcp_planner_ucp_rr(dcp_planner* pl, int32_t* rr, int32_t n, int32_t dir) {
    DCP_REQUIRE(pl && (n == 0 || rr) && n >= 0 && (dir == 0 || dir == 1), DCP_E_INVALID_ARG, "bad argument");
    PlannerState& st = pl->st;
    if (dir == 0) {
        if (n != st.n_groups || !st.ucp_rr) {
            if (st.ucp_rr) {
                DCP_CUDA_TRY(cudaFree(st.ucp_rr));
                auto it = std::find(pl->owned.begin(), pl->owned.end(), static_cast<void*>(st.ucp_rr));
                if (it != pl->owned.end()) pl->owned.erase(it);
            }
            void* q = nullptr;
            DCP_CUDA_TRY(cudaMalloc(&q, std::max(n, 1) * sizeof(int32_t)));
            pl->owned.push_back(q);
            st.ucp_rr = static_cast<int32_t*>(q);
            st.n_groups = n;
        }
        if (n) DCP_CUDA_TRY(cudaMemcpy(st.ucp_rr, rr, n * sizeof(int32_t), cudaMemcpyHostToDevice));
    } else {
        DCP_REQUIRE(n == st.n_groups, DCP_E_INVALID_ARG, "rr size %d != %d groups", n, st.n_groups);
        if (n) DCP_CUDA_TRY(cudaMemcpy(rr, st.ucp_rr, n * sizeof(int32_t), cudaMemcpyDeviceToHost));
    }
    return DCP_OK;
}

int dcp_planner_set_queue(dcp_planner* pl, const int64_t* ids, const int64_t* lens, int32_t n) {
    DCP_REQUIRE(pl && (n == 0 || (ids && lens)), DCP_E_INVALID_ARG, "NULL argument");
    std::vector<int32_t> state;
    if (int rc = planner_states(pl, state)) return rc;
    std::vector<int32_t> slots(n), is_new(n, 0), drop;
    std::unordered_map<int64_t, int> listed;
    for (int i = 0; i < n; ++i) listed[ids[i]] = i;
    DCP_REQUIRE((int)listed.size() == n, DCP_E_INVALID_ARG, "duplicate id in waiting queue");
    // waiting requests no longer listed are dropped
    for (auto it = pl->slot_of.begin(); it != pl->slot_of.end();) {
        if (state[it->second] == ST_WAITING && !listed.count(it->first)) {
            drop.push_back(it->second);
            pl->free_slots.push_back(it->second);
            pl->id_of_slot[it->second] = -1;
            it = pl->slot_of.erase(it);
        } else {
            ++it;
        }
    }
    int64_t bound = 0;
    for (int i = 0; i < n; ++i) {
        auto it = pl->slot_of.find(ids[i]);
        if (it != pl->slot_of.end()) {
            DCP_REQUIRE(state[it->second] == ST_WAITING, DCP_E_INSUFFICIENT_FRAMES,
                        "request %lld already has page-table entries", (long long)ids[i]);
            slots[i] = it->second;
        } else {
            DCP_REQUIRE(!pl->free_slots.empty(), DCP_E_INVALID_ARG, "request slots exhausted");
            const int sl = pl->free_slots.back();
            pl->free_slots.pop_back();
            pl->slot_of[ids[i]] = sl;
            pl->id_of_slot[sl] = ids[i];
            pl->retired.erase(ids[i]);
            slots[i] = sl;
            is_new[i] = 1;
        }
        pl->queued_len[slots[i]] = lens[i];
        bound += (lens[i] + pl->cfg.page_size - 1) / pl->cfg.page_size + PL_MAXK + pl->st.reserve_pages;
    }
    pl->queued = n;
    pl->waiting_pages_bound = bound;
    TmpFree tf;
    int32_t *d_slots, *d_new, *d_drop;
    int64_t *d_ids, *d_lens;
    int rc = 0;
    rc |= dalloc_tmp(&d_slots, n, tf.v);
    rc |= dalloc_tmp(&d_new, n, tf.v);
    rc |= dalloc_tmp(&d_drop, drop.size(), tf.v);
    rc |= dalloc_tmp(&d_ids, n, tf.v);
    rc |= dalloc_tmp(&d_lens, n, tf.v);
    if (rc) return DCP_E_CUDA;
    if (n) {
        DCP_CUDA_TRY(cudaMemcpy(d_slots, slots.data(), n * 4, cudaMemcpyHostToDevice));
        DCP_CUDA_TRY(cudaMemcpy(d_new, is_new.data(), n * 4, cudaMemcpyHostToDevice));
        DCP_CUDA_TRY(cudaMemcpy(d_ids, ids, n * 8, cudaMemcpyHostToDevice));
        DCP_CUDA_TRY(cudaMemcpy(d_lens, lens, n * 8, cudaMemcpyHostToDevice));
    }
    if (!drop.empty()) DCP_CUDA_TRY(cudaMemcpy(d_drop, drop.data(), drop.size() * 4, cudaMemcpyHostToDevice));
    set_queue_kernel<<<1, 256, 0, pl->stream>>>(pl->st, d_slots, d_ids, d_lens, d_new, n, d_drop,
                                                (int)drop.size());
    DCP_CUDA_TRY(cudaGetLastError());
    DCP_CUDA_TRY(cudaStreamSynchronize(pl->stream));
    return DCP_OK;
}

int dcp_planner_allocate(dcp_planner* pl, int64_t id, int64_t seq_len, int32_t k, const int32_t* kv,
                         const int64_t* split, int32_t moe) {
    DCP_REQUIRE(pl && kv && split, DCP_E_INVALID_ARG, "NULL argument");
    DCP_REQUIRE(k >= 1 && k <= PL_MAXK, DCP_E_UNSUPPORTED, "cp_degree %d", k);
    for (int m = 0; m < k; ++m) {
        DCP_REQUIRE(kv[m] >= 0 && kv[m] < pl->st.W, DCP_E_INVALID_ARG, "instance %d out of range", kv[m]);
        // the device allocator pops every member's frames from the same pre-pop stack top
        for (int j = 0; j < m; ++j)
            DCP_REQUIRE(kv[j] != kv[m], DCP_E_INCONSISTENT, "instance %d listed twice in kv_binding", kv[m]);
    }
    std::vector<int32_t> state;
    if (int rc = planner_states(pl, state)) return rc;
    int sl;
    bool fresh = false;
    auto it = pl->slot_of.find(id);
    if (it != pl->slot_of.end()) {
        DCP_REQUIRE(state[it->second] != ST_ACTIVE, DCP_E_INSUFFICIENT_FRAMES,
                    "request already has page-table entries");
        sl = it->second;
    } else {
        DCP_REQUIRE(!pl->free_slots.empty(), DCP_E_INVALID_ARG, "request slots exhausted");
        sl = pl->free_slots.back();
        pl->free_slots.pop_back();
        fresh = true;
    }
    int64_t np = 0;
    for (int m = 0; m < k; ++m) np += (split[m] + pl->cfg.page_size - 1) / pl->cfg.page_size;
    if (pl->arena_top_host + np + pl->st.reserve_pages > pl->st.arena_cap)
        if (int rc = planner_compact(pl)) return rc;
    TmpFree tf;
    int32_t* d_kv;
    int64_t* d_split;
    if (dalloc_tmp(&d_kv, k, tf.v) || dalloc_tmp(&d_split, k, tf.v)) return DCP_E_CUDA;
    DCP_CUDA_TRY(cudaMemcpy(d_kv, kv, k * 4, cudaMemcpyHostToDevice));
    DCP_CUDA_TRY(cudaMemcpy(d_split, split, k * 8, cudaMemcpyHostToDevice));
    const int32_t st_w = ST_WAITING;
    DCP_CUDA_TRY(cudaMemcpy(pl->st.id + sl, &id, 8, cudaMemcpyHostToDevice));
    DCP_CUDA_TRY(cudaMemcpy(pl->st.seq_len + sl, &seq_len, 8, cudaMemcpyHostToDevice));
    if (fresh) DCP_CUDA_TRY(cudaMemcpy(pl->st.state + sl, &st_w, 4, cudaMemcpyHostToDevice));
    planner_allocate_kernel<<<1, PL_THREADS, 0, pl->stream>>>(pl->st, sl, k, d_kv, d_split, moe);
    DCP_CUDA_TRY(cudaGetLastError());
    DCP_CUDA_TRY(cudaStreamSynchronize(pl->stream));
    int32_t cnt[4];
    DCP_CUDA_TRY(cudaMemcpy(cnt, pl->st.res_counts, sizeof(cnt), cudaMemcpyDeviceToHost));
    if (cnt[3] != PL_OK) {
        if (fresh) {
            const int32_t st_f = ST_FREE;
            DCP_CUDA_TRY(cudaMemcpy(pl->st.state + sl, &st_f, 4, cudaMemcpyHostToDevice));
            pl->free_slots.push_back(sl);
        }
        set_error(cnt[3] == PL_E_FRAMES ? "instance lacks frames for request %lld"
                                        : "page arena exhausted for request %lld",
                  (long long)id);
        return cnt[3] == PL_E_FRAMES ? DCP_E_INSUFFICIENT_FRAMES : DCP_E_CUDA;
    }
    if (fresh) {
        pl->slot_of[id] = sl;
        pl->id_of_slot[sl] = id;
        pl->retired.erase(id);
    }
    pl->is_active[sl] = 1;
    pl->routing_valid = false;
    return planner_sync_arena_top(pl);
}

int64_t dcp_planner_pages(dcp_planner* pl, int64_t id, int32_t* inst, int32_t* frame, int64_t cap) {
    if (!pl) return DCP_E_INVALID_ARG;
    auto it = pl->slot_of.find(id);
    if (it == pl->slot_of.end()) {
        set_error("unknown request %lld", (long long)id);
        return DCP_E_UNKNOWN_REQUEST;
    }
    const int sl = it->second;
    if (cudaStreamSynchronize(pl->stream) != cudaSuccess) return DCP_E_CUDA;
    int32_t state = 0, cnt = 0;
    int64_t off = 0;
    cudaMemcpy(&state, pl->st.state + sl, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&cnt, pl->st.page_cnt + sl, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&off, pl->st.page_off + sl, 8, cudaMemcpyDeviceToHost);
    if (state != ST_ACTIVE) {
        set_error("no page-table entries for request %lld", (long long)id);
        return DCP_E_UNKNOWN_REQUEST;
    }
    const int64_t n = std::min<int64_t>(cnt, cap);
    if (n > 0 && inst) cudaMemcpy(inst, pl->st.pg_inst + off, n * 4, cudaMemcpyDeviceToHost);
    if (n > 0 && frame) cudaMemcpy(frame, pl->st.pg_frame + off, n * 4, cudaMemcpyDeviceToHost);
    if (cudaGetLastError() != cudaSuccess) return DCP_E_CUDA;
    return cnt;
}

int32_t dcp_planner_active_moe(dcp_planner* pl, int64_t* ids, int32_t* moe, int32_t cap) {
    if (!pl) return DCP_E_INVALID_ARG;
    std::vector<int32_t> state;
    if (int rc = planner_states(pl, state)) return rc;
    const size_t S = pl->cfg.max_requests;
    std::vector<int32_t> m(S);
    std::vector<int64_t> id(S);
    cudaMemcpy(m.data(), pl->st.moe, S * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(id.data(), pl->st.id, S * 8, cudaMemcpyDeviceToHost);
    if (cudaGetLastError() != cudaSuccess) return DCP_E_CUDA;
    int32_t n = 0;
    for (size_t s = 0; s < S; ++s)
        if (state[s] == ST_ACTIVE) {
            if (n < cap) {
                ids[n] = id[s];
                moe[n] = m[s];
            }
            ++n;
        }
    return n;
}

int dcp_planner_rebalance(dcp_planner* pl, const int64_t* ids, int32_t n) {
    DCP_REQUIRE(pl && (n == 0 || ids), DCP_E_INVALID_ARG, "NULL argument");
    std::vector<int32_t> state;
    if (int rc = planner_states(pl, state)) return rc;
    std::vector<int32_t> slots(n);
    for (int i = 0; i < n; ++i) {
        auto it = pl->slot_of.find(ids[i]);
        DCP_REQUIRE(it != pl->slot_of.end() && state[it->second] == ST_ACTIVE, DCP_E_UNKNOWN_REQUEST,
                    "request %lld has no placement", (long long)ids[i]);
        slots[i] = it->second;
    }
    TmpFree tf;
    int32_t* d;
    if (dalloc_tmp(&d, n, tf.v)) return DCP_E_CUDA;
    if (n) DCP_CUDA_TRY(cudaMemcpy(d, slots.data(), n * 4, cudaMemcpyHostToDevice));
    planner_rebalance_kernel<<<1, PL_THREADS, 0, pl->stream>>>(pl->st, d, n);
    DCP_CUDA_TRY(cudaGetLastError());
    DCP_CUDA_TRY(cudaStreamSynchronize(pl->stream));
    pl->routing_valid = false;
    return DCP_OK;
}

int dcp_planner_load_instances(dcp_planner* pl, const int64_t* kv, const int32_t* b, const int32_t* sc,
                               const int64_t* nf, const int32_t* stacks) {
    DCP_REQUIRE(pl && kv && b && sc && nf && stacks, DCP_E_INVALID_ARG, "NULL argument");
    DCP_REQUIRE(pl->slot_of.empty(), DCP_E_INVALID_ARG, "planner must be idle to load instance state");
    const int W = pl->st.W;
    const size_t tot = (size_t)W * pl->st.capacity;
    TmpFree tf;
    int64_t *dkv, *dnf;
    int32_t *db, *dsc, *dst;
    int rc = dalloc_tmp(&dkv, W, tf.v) | dalloc_tmp(&dnf, W, tf.v) | dalloc_tmp(&db, W, tf.v) |
             dalloc_tmp(&dsc, W, tf.v) | dalloc_tmp(&dst, tot, tf.v);
    if (rc) return DCP_E_CUDA;
    for (int s = 0; s < W; ++s)
        DCP_REQUIRE(nf[s] >= 0 && nf[s] <= pl->st.capacity, DCP_E_INVALID_ARG, "free count out of range");
    DCP_CUDA_TRY(cudaMemcpy(dkv, kv, W * 8, cudaMemcpyHostToDevice));
    DCP_CUDA_TRY(cudaMemcpy(dnf, nf, W * 8, cudaMemcpyHostToDevice));
    DCP_CUDA_TRY(cudaMemcpy(db, b, W * 4, cudaMemcpyHostToDevice));
    DCP_CUDA_TRY(cudaMemcpy(dsc, sc, W * 4, cudaMemcpyHostToDevice));
    if (tot) DCP_CUDA_TRY(cudaMemcpy(dst, stacks, tot * 4, cudaMemcpyHostToDevice));
    load_instances_kernel<<<64, 256, 0, pl->stream>>>(pl->st, dkv, db, dsc, dnf, dst);
    DCP_CUDA_TRY(cudaGetLastError());
    DCP_CUDA_TRY(cudaStreamSynchronize(pl->stream));
    return DCP_OK;
}

int dcp_water_fill(dcp_ctx* ctx, int32_t n, const int64_t* loads, int64_t seq_len, int64_t* split) {
    DCP_REQUIRE(ctx && loads && split, DCP_E_INVALID_ARG, "NULL argument");
    DCP_REQUIRE(n >= 1 && n <= 32, DCP_E_UNSUPPORTED, "water_fill over %d participants (<=32)", n);
    TmpFree tf;
    int64_t *dl, *ds;
    if (dalloc_tmp(&dl, n, tf.v) || dalloc_tmp(&ds, n, tf.v)) return DCP_E_CUDA;
    DCP_CUDA_TRY(cudaMemcpy(dl, loads, n * 8, cudaMemcpyHostToDevice));
    water_fill_kernel<<<1, 32>>>(n, dl, seq_len, ds);
    DCP_CUDA_TRY(cudaGetLastError());
    DCP_CUDA_TRY(cudaMemcpy(split, ds, n * 8, cudaMemcpyDeviceToHost));
    return DCP_OK;
}

int dcp_binding_config(dcp_ctx* ctx, int32_t n, const int64_t* ids, const int32_t* k, const int32_t* moe,
                       const int32_t* kv, int32_t W, int32_t* n_count, int32_t* m_count, int32_t* n_rows,
                       int32_t* m_rows) {
    DCP_REQUIRE(ctx && n_count && m_count, DCP_E_INVALID_ARG, "NULL argument");
    DCP_REQUIRE(W >= 1 && W <= PL_MAXW, DCP_E_UNSUPPORTED, "world %d", W);
    if (n == 0) {
        for (int s = 0; s < W; ++s) n_count[s] = m_count[s] = 0;
        return DCP_OK;
    }
    DCP_REQUIRE(ids && k && moe && kv && n_rows && m_rows, DCP_E_INVALID_ARG, "NULL argument");
    for (int i = 0; i < n; ++i) {
        DCP_REQUIRE(k[i] >= 1 && k[i] <= PL_MAXK, DCP_E_UNSUPPORTED, "cp_degree %d", k[i]);
        for (int m = 0; m < k[i]; ++m)
            DCP_REQUIRE(kv[i * PL_MAXK + m] >= 0 && kv[i * PL_MAXK + m] < W, DCP_E_INVALID_ARG,
                        "kv_binding instance out of range");
    }
    DCP_REQUIRE(moe != nullptr, DCP_E_INVALID_ARG, "NULL moe");
    TmpFree tf;
    PlannerState st{};
    RoutingOut ro{};
    st.W = W;
    st.max_slots = n;
    int sort_cap = 1;
    while (sort_cap < n) sort_cap <<= 1;
    st.sort_cap = sort_cap;
    std::vector<int32_t> active(n, ST_ACTIVE);
    int rc = 0;
    rc |= dalloc_tmp(&st.state, n, tf.v);
    rc |= dalloc_tmp(&st.id, n, tf.v);
    rc |= dalloc_tmp(&st.k, n, tf.v);
    rc |= dalloc_tmp(&st.moe, n, tf.v);
    rc |= dalloc_tmp(&st.kv, (size_t)n * PL_MAXK, tf.v);
    rc |= dalloc_tmp(&st.shard_tokens, (size_t)n * W, tf.v);
    rc |= dalloc_tmp(&st.last_append, n, tf.v);
    rc |= dalloc_tmp(&st.sk1, sort_cap, tf.v);
    rc |= dalloc_tmp(&st.sk2, sort_cap, tf.v);
    rc |= dalloc_tmp(&st.sval, sort_cap, tf.v);
    rc |= dalloc_tmp(&ro.n_count, W, tf.v);
    rc |= dalloc_tmp(&ro.m_count, W, tf.v);
    rc |= dalloc_tmp(&ro.n_id, (size_t)W * n, tf.v);
    rc |= dalloc_tmp(&ro.n_slot, (size_t)W * n, tf.v);
    rc |= dalloc_tmp(&ro.n_moe, (size_t)W * n, tf.v);
    rc |= dalloc_tmp(&ro.q_route, (size_t)W * n * W, tf.v);
    rc |= dalloc_tmp(&ro.m_id, (size_t)W * n, tf.v);
    rc |= dalloc_tmp(&ro.m_slot, (size_t)W * n, tf.v);
    rc |= dalloc_tmp(&ro.res_route, (size_t)W * n * W, tf.v);
    rc |= dalloc_tmp(&ro.bucket, 2 * W, tf.v);
    rc |= dalloc_tmp(&ro.shard_len, (size_t)W * n, tf.v);
    rc |= dalloc_tmp(&ro.slot_nrow, (size_t)n * W, tf.v);
    rc |= dalloc_tmp(&ro.slot_mrow, n, tf.v);
    rc |= dalloc_tmp(&ro.status, 1, tf.v);
    rc |= dalloc_tmp(&ro.n_active, 1, tf.v);
    if (rc) return DCP_E_CUDA;
    DCP_CUDA_TRY(cudaMemcpy(st.state, active.data(), n * 4, cudaMemcpyHostToDevice));
    DCP_CUDA_TRY(cudaMemcpy(st.id, ids, n * 8, cudaMemcpyHostToDevice));
    DCP_CUDA_TRY(cudaMemcpy(st.k, k, n * 4, cudaMemcpyHostToDevice));
    DCP_CUDA_TRY(cudaMemcpy(st.moe, moe, n * 4, cudaMemcpyHostToDevice));
    DCP_CUDA_TRY(cudaMemcpy(st.kv, kv, (size_t)n * PL_MAXK * 4, cudaMemcpyHostToDevice));
    DCP_CUDA_TRY(launch_routing_rows(st, ro, nullptr));
    DCP_CUDA_TRY(cudaGetLastError());
    int32_t status = 0;
    DCP_CUDA_TRY(cudaMemcpy(&status, ro.status, 4, cudaMemcpyDeviceToHost));
    DCP_REQUIRE(status == 0, DCP_E_INCONSISTENT, "moe_binding outside kv_binding");
    DCP_CUDA_TRY(cudaMemcpy(n_count, ro.n_count, W * 4, cudaMemcpyDeviceToHost));
    DCP_CUDA_TRY(cudaMemcpy(m_count, ro.m_count, W * 4, cudaMemcpyDeviceToHost));
    DCP_CUDA_TRY(cudaMemcpy(n_rows, ro.n_slot, (size_t)W * n * 4, cudaMemcpyDeviceToHost));
    DCP_CUDA_TRY(cudaMemcpy(m_rows, ro.m_slot, (size_t)W * n * 4, cudaMemcpyDeviceToHost));
    return DCP_OK;
}

int dcp_route_tables(dcp_ctx* ctx, int32_t W, int32_t n, const int32_t* shard_moe, int32_t m,
                     const uint32_t* res_mask, uint8_t* q_bits, uint8_t* res_bits) {
    DCP_REQUIRE(ctx && (n == 0 || (shard_moe && q_bits)) && (m == 0 || (res_mask && res_bits)),
                DCP_E_INVALID_ARG, "NULL argument");
    DCP_REQUIRE(W >= 1 && W <= 32, DCP_E_UNSUPPORTED, "world %d", W);
    if (n == 0 && m == 0) return DCP_OK;
    TmpFree tf;
    int32_t* d_sm;
    uint32_t* d_rm;
    uint8_t *dq, *dr;
    if (dalloc_tmp(&d_sm, n, tf.v) || dalloc_tmp(&d_rm, m, tf.v) || dalloc_tmp(&dq, (size_t)n * W, tf.v) ||
        dalloc_tmp(&dr, (size_t)m * W, tf.v))
        return DCP_E_CUDA;
    if (n) DCP_CUDA_TRY(cudaMemcpy(d_sm, shard_moe, n * 4, cudaMemcpyHostToDevice));
    if (m) DCP_CUDA_TRY(cudaMemcpy(d_rm, res_mask, m * 4, cudaMemcpyHostToDevice));
    route_expand_kernel<<<64, 256>>>(W, n, d_sm, m, d_rm, dq, dr);
    DCP_CUDA_TRY(cudaGetLastError());
    if (n) DCP_CUDA_TRY(cudaMemcpy(q_bits, dq, (size_t)n * W, cudaMemcpyDeviceToHost));
    if (m) DCP_CUDA_TRY(cudaMemcpy(res_bits, dr, (size_t)m * W, cudaMemcpyDeviceToHost));
    return DCP_OK;
}

int dcp_shard_attention_batch(dcp_ctx* ctx, int32_t dtype_bytes, int32_t n, int32_t d, double scale,
                              const void* q, const void* keys, const void* values, const int64_t* q_off,
                              const int64_t* kv_off, const int64_t* len, void* out, void* lse, void* stream) {
    DCP_REQUIRE(ctx && q && keys && values && q_off && kv_off && len && out && lse, DCP_E_INVALID_ARG,
                "NULL argument");
    DCP_REQUIRE(d >= 1 && d <= CONTIG_MAXD, DCP_E_UNSUPPORTED, "head_dim %d (<= %d)", d, CONTIG_MAXD);
    if (n <= 0) return DCP_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (dtype_bytes == 4) {
        shard_attn_contig_kernel<float><<<n, 128, 0, s>>>(
            d, (float)scale, static_cast<const float*>(q), static_cast<const float*>(keys),
            static_cast<const float*>(values), q_off, kv_off, len, static_cast<float*>(out), static_cast<float*>(lse));
    } else if (dtype_bytes == 8) {
        shard_attn_contig_kernel<double><<<n, 128, 0, s>>>(
            d, scale, static_cast<const double*>(q), static_cast<const double*>(keys),
            static_cast<const double*>(values), q_off, kv_off, len, static_cast<double*>(out),
            static_cast<double*>(lse));
    } else {
        set_error("dtype_bytes %d (4 or 8)", dtype_bytes);
        return DCP_E_UNSUPPORTED;
    }
    DCP_CUDA_TRY(cudaGetLastError());
    return DCP_OK;
}

int dcp_lse_merge_batch(dcp_ctx* ctx, int32_t dtype_bytes, int32_t g, int32_t d, const int64_t* off,
                        const void* outs, const void* lses, void* merged, void* merged_lse, void* stream) {
    DCP_REQUIRE(ctx && off && outs && lses && merged, DCP_E_INVALID_ARG, "NULL argument");
    if (g <= 0) return DCP_OK;
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (dtype_bytes == 4)
        lse_merge_contig_kernel<float><<<g, 128, 0, s>>>(d, off, static_cast<const float*>(outs),
                                                         static_cast<const float*>(lses), static_cast<float*>(merged),
                                                         static_cast<float*>(merged_lse));
    else if (dtype_bytes == 8)
        lse_merge_contig_kernel<double><<<g, 128, 0, s>>>(d, off, static_cast<const double*>(outs),
                                                          static_cast<const double*>(lses),
                                                          static_cast<double*>(merged), static_cast<double*>(merged_lse));
    else {
        set_error("dtype_bytes %d (4 or 8)", dtype_bytes);
        return DCP_E_UNSUPPORTED;
    }
    DCP_CUDA_TRY(cudaGetLastError());
    return DCP_OK;
}

}  // extern "C"
