// SPDX-License-Identifier: Apache-2.0
//
// K6: the DCP planner as device kernels (north_star subsystem 4).
//
// Restates, bit-exactly, the integer control plane of the reference:
//   Scheduler::step            scheduler.cpp:245-306  (FIFO admission, HoL counting)
//   rebalance_active           scheduler.cpp:43-64    (Alg. 1 lines 1-5)
//   place_dcp / min_batch      scheduler.cpp:118-170  (Alg. 1 lines 7-12)
//   place_single               scheduler.cpp:172-187  (LeastBatch / LeastCache)
//   place_uniform              scheduler.cpp:189-223  (UniformCP, round-robin m_r)
//   never_fits / can_allocate  scheduler.cpp:225-243, 104-113
//   water_fill                 scheduler.cpp:70-102
//   cp_degree / BucketFn       scheduler.cpp:10-33, 66-68
//   GlobalPageTable::allocate / release / append_token   page_table.cpp:9-121
//   make_cluster LIFO stacks   page_table.cpp:133-148
//
// The admission loop is inherently sequential (each commit mutates the K/B/
// free-frame state the next request reads), so it runs in ONE CTA: instance
// state lives in shared memory, warp 0 makes each decision with one lane per
// instance (warp argmin / rank / ballot replace the reference's loops and
// std::stable_sort), and the whole CTA copies the popped frame ids.  Rebalance
// exploits the (cp_degree, id) order: all CP=1 requests come first and pin
// m_r to their single instance (a parallel histogram), only CP>=2 requests
// need the sequential argmin.
#pragma once

#include <cstdint>

#include "limits.cuh"
#include "ptx.cuh"

namespace dcp {

constexpr int PL_THREADS = 512;

enum : int32_t { PL_OK = 0, PL_E_FRAMES = -1, PL_E_UNKNOWN = -2, PL_E_ARENA = -11 };
enum : int32_t { KIND_DCP = 0, KIND_LEAST_BATCH = 1, KIND_LEAST_CACHE = 2, KIND_UNIFORM = 3 };
enum : int32_t { ST_WAITING = 0, ST_ACTIVE = 1, ST_FINISHED = 2, ST_FREE = 3 };

struct PlannerState {
    // ---- configuration
    int32_t nodes, ipn, W, kind, udeg, hol_strict, nbucket, max_slots;
    int64_t page, capacity, arena_cap, reserve_pages;
    int64_t bucket_len[16];
    int32_t bucket_deg[16];
    int32_t n_groups;
    // ---- instance state (InstanceState, page_table.hpp:13-25)
    int64_t* kv_load;      // [W]  K_s
    int32_t* moe_batch;    // [W]  B_s
    int32_t* shard_count;  // [W]  R_i
    int64_t* nfree;        // [W]  |free_frames|
    int32_t* stack;        // [W][capacity] LIFO, top at nfree-1
    int32_t* ucp_rr;       // [n_groups] UniformCP round robin (scheduler.hpp:88)
    // ---- request slots (Request + Placement + GlobalPageTable::Entry)
    int64_t* id;
    int64_t* seq_len;
    int64_t* generated;
    int32_t* state;
    int32_t* k;
    int32_t* moe;
    int32_t* kv;           // [S][PL_MAXK]
    int64_t* split;        // [S][PL_MAXK]
    int64_t* page_off;     // [S] segment start in the page arena
    int32_t* page_cnt;     // [S]
    int32_t* page_cap;     // [S]
    int64_t* trailing_fill;// [S]
    int64_t* shard_tokens; // [S][W]
    int32_t* last_append;  // [S] instance that received the latest append_token, -1 = stall
    int32_t* pg_inst;      // arena [arena_cap]
    int32_t* pg_frame;     // arena
    uint8_t* pg_fill;      // arena: valid tokens of each page
    int64_t* arena_top;    // [1]
    // ---- waiting queue (deque<size_t>) of slots
    int32_t* waiting;      // [S]
    int32_t* nwait;        // [1]
    // ---- step results (StepResult, scheduler.hpp:58-65)
    int32_t* res_slots;    // [3][S]: committed, deferred, unschedulable (slot ids)
    int32_t* res_counts;   // [4]: n_committed, n_deferred, n_unsched, status
    int64_t* res_hol;      // [1]
    struct PageRec* recs;  // [S] frame pops of the step's commits, in commit order
    int64_t* res_pages;    // [1] pages popped by the step (sum over recs)
    // ---- scratch
    int64_t* sk1;          // [sort_cap]
    int64_t* sk2;
    int32_t* sval;
    int32_t sort_cap;
};

// ------------------------------------------------------------------ warp helpers
__device__ __forceinline__ int64_t warp_sum_i64(int64_t v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ int64_t warp_max_i64(int64_t v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const int64_t u = __shfl_xor_sync(0xffffffffu, v, o);
        v = u > v ? u : v;
    }
    return v;
}
// argmin of (value) with ties to the lowest index; returns the winning index.
__device__ __forceinline__ int warp_argmin_i64(int64_t v, int idx) {
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        const int64_t ov = __shfl_xor_sync(0xffffffffu, v, o);
        const int oi = __shfl_xor_sync(0xffffffffu, idx, o);
        if (ov < v || (ov == v && oi < idx)) { v = ov; idx = oi; }
    }
    return idx;
}

// argmin over lanes of small non-negative counts (< 2^22, the B_s batch counts and their node
// sums; dcp_planner_create bounds max_requests), ties to the lowest lane: one redux.sync on the
// packed key (value, lane) instead of five shuffle rounds.
__device__ __forceinline__ int warp_argmin_small(uint32_t v, bool valid, int lane) {
    const uint32_t key = valid ? (v << 5) | static_cast<uint32_t>(lane) : 0xffffffffu;
    return static_cast<int>(__reduce_min_sync(0xffffffffu, key) & 31u);
}

// ceil(tokens / page) (types.hpp:100-102); a power-of-two page (16 by default) takes a shift
// instead of a 64-bit division, which is a ~100-instruction call on the admission path.
__device__ __forceinline__ int64_t pages_for_d(int64_t tokens, int64_t page) {
    if ((page & (page - 1)) == 0) return (tokens + page - 1) >> (__ffsll(page) - 1);
    return (tokens + page - 1) / page;
}
__device__ __forceinline__ int64_t page_rem_d(int64_t tokens, int64_t page) {
    if ((page & (page - 1)) == 0) return tokens & (page - 1);
    return tokens % page;
}

__device__ __forceinline__ int bucket_lookup_d(const PlannerState& st, int64_t len) {
    for (int i = 0; i < st.nbucket; ++i)
        if (len <= st.bucket_len[i]) return st.bucket_deg[i];
    return st.bucket_deg[st.nbucket - 1];
}
__device__ __forceinline__ int cp_degree_d(const PlannerState& st, int64_t len) {
    const int d = bucket_lookup_d(st, len);
    return d < st.ipn ? d : st.ipn;
}

// Shared-memory image of the instance state during a step.
struct SmemInst {
    int64_t K[PL_MAXW];
    int64_t nfree[PL_MAXW];
    int32_t B[PL_MAXW];
    int32_t shards[PL_MAXW];
};

struct SmemPlace {
    int32_t k, moe;
    int32_t kv[PL_MAXK];
    int64_t split[PL_MAXK];
    int64_t need_off[PL_MAXK + 1];  // page prefix over members
    int32_t ok;                     // can_allocate
    int32_t unsched;
};

// One commit: its frame pops and its slot fields.  Warp 0 of the step records it; planner_pages_kernel
// writes the slot's placement / page-table fields and copies the popped frame ids afterwards.
struct alignas(16) PageRec {
    int64_t base;                   // pages of the step's earlier commits
    int64_t off;                    // arena segment start
    int32_t k, sl, moe, cap;        // members, slot, m_r, reserved pages of the segment
    int32_t kv[PL_MAXK];
    int64_t top[PL_MAXK];           // nfree of each member before the pops
    int64_t split[PL_MAXK];
    int64_t need_off[PL_MAXK + 1];
};

// water_fill (scheduler.cpp:70-102) with one lane per participant (lanes < n).
// The level -- the minimal integer P with sum_i max(0, P - K_i) >= len, which the reference
// finds by binary search (cpp:74-86) -- is computed in closed form: with the K_i sorted
// ascending, the first j whose candidate P_j = ceil((len + K_(0) + .. + K_(j-1)) / j) does not
// exceed K_(j) (or j = n) is the piece of the convex f(P) where f first reaches len.  Same
// integer, no ~log2(K + len) warp reductions.
__device__ __forceinline__ int64_t warp_water_fill(int lane, int n, int64_t len, int64_t K) {
    const bool part = lane < n;
    int64_t level;
    if (n == 1) {
        level = __shfl_sync(0xffffffffu, K, 0) + len;
    } else {
        int64_t ks[32];  // n <= 32 (dcp_water_fill); the planner uses n <= instances_per_node <= 16
        int m = 0;
        for (int j = 0; j < n; ++j) {  // every lane: the participants' K, insertion-sorted
            const int64_t v = __shfl_sync(0xffffffffu, K, j);
            int i = m++;
            while (i > 0 && ks[i - 1] > v) {
                ks[i] = ks[i - 1];
                --i;
            }
            ks[i] = v;
        }
        int64_t prefix = 0;
        level = 0;
        for (int j = 1; j <= n; ++j) {
            prefix += ks[j - 1];
            const int64_t pj = (len + prefix + j - 1) / j;
            if (j == n || pj <= ks[j]) {
                level = pj;
                break;
            }
        }
    }
    int64_t s = part && level - 1 - K > 0 ? level - 1 - K : 0;
    const int64_t rem = len - warp_sum_i64(s);
    const bool elig = part && (K + s < level);
    const unsigned bal = __ballot_sync(0xffffffffu, elig);
    const int rank = __popc(bal & ((1u << lane) - 1u));
    if (elig && rank < rem) s += 1;
    return s;
}

// Placement decision for one request (warp 0).  Writes *pl.
static __device__ void place_request(const PlannerState& st, const SmemInst& si, SmemPlace& pl, int lane,
                              int64_t L, int k_dcp) {
    const int W = st.W, ipn = st.ipn;
    if (st.kind == KIND_DCP) {
        // node = argmin_n sum_{s in n} B_s, ties by node id (scheduler.cpp:133-141)
        uint32_t bn = 0;
        if (lane < st.nodes)
            for (int s = lane * ipn; s < (lane + 1) * ipn; ++s) bn += si.B[s];
        const int node = st.nodes == 1 ? 0 : warp_argmin_small(bn, lane < st.nodes, lane);
        const int k = k_dcp;
        const int nb = node * ipn;
        // m_r = min_batch_instance over the node, ties to lowest id (cpp:118-126)
        const int moe = nb + warp_argmin_small(lane < ipn ? si.B[nb + lane] : 0u, lane < ipn, lane);
        if (k == 1) {  // P_r = [m_r], water_fill of one participant = the whole request, can_allocate
            if (lane == 0) {
                const int64_t need = pages_for_d(L, st.page);
                pl.kv[0] = moe;
                pl.moe = moe;
                pl.k = 1;
                pl.split[0] = L;
                pl.need_off[0] = 0;
                pl.need_off[1] = need;
                pl.ok = si.nfree[moe] >= need ? 1 : 0;
            }
            __syncwarp();
            return;
        }
        // SelectSmallestKV: node minus m_r by (K, id) (cpp:148-156) -> rank per lane
        if (lane < ipn) {
            const int s = nb + lane;
            if (s != moe) {
                int rank = 0;
                for (int j = nb; j < nb + ipn; ++j) {
                    if (j == moe || j == s) continue;
                    if (si.K[j] < si.K[s] || (si.K[j] == si.K[s] && j < s)) ++rank;
                }
                if (rank < k - 1) pl.kv[1 + rank] = s;
            }
        }
        if (lane == 0) {
            pl.kv[0] = moe;
            pl.moe = moe;
            pl.k = k;
        }
        __syncwarp();
        if (k == 1) {  // water_fill over one participant: the whole request (cpp:70-102)
            if (lane == 0) pl.split[0] = L;
        } else {
            const int64_t Kl = lane < k ? si.K[pl.kv[lane]] : 0;
            const int64_t s = warp_water_fill(lane, k, L, Kl);
            if (lane < k) pl.split[lane] = s;
        }
    } else if (st.kind == KIND_LEAST_BATCH || st.kind == KIND_LEAST_CACHE) {
        // argmin over all instances, first minimum (cpp:172-187)
        int64_t v = INT64_MAX;
        if (lane < W) v = st.kind == KIND_LEAST_BATCH ? (int64_t)si.B[lane] : si.K[lane];
        const int best = warp_argmin_i64(v, lane);
        if (lane == 0) {
            pl.k = 1;
            pl.moe = best;
            pl.kv[0] = best;
            pl.split[0] = L;
        }
    } else {
        // UniformCP (cpp:189-223): group with fewest MoE-bound requests
        const int d = st.udeg;
        int64_t bg = INT64_MAX;
        if (lane < st.n_groups) {
            bg = 0;
            for (int s = lane * d; s < lane * d + d; ++s) bg += si.B[s];
        }
        const int g = warp_argmin_i64(bg, lane);
        const int gb = g * d;
        if (lane < d) {
            const int64_t base = L / d;
            const int64_t rem = L % d;
            pl.kv[lane] = gb + lane;
            pl.split[lane] = base + (lane < rem ? 1 : 0);
        }
        if (lane == 0) {
            pl.k = d;
            const int rr = st.ucp_rr[g];
            pl.moe = gb + rr;
            st.ucp_rr[g] = (rr + 1) % d;  // advanced even if the request is deferred
        }
    }
    __syncwarp();
    // can_allocate (cpp:104-113) + page prefix for the allocation
    const int k = pl.k;
    int64_t need = 0;
    bool ok = true;
    if (lane < k) {
        need = pages_for_d(pl.split[lane], st.page);
        ok = si.nfree[pl.kv[lane]] >= need;
    }
    const bool all_ok = __all_sync(0xffffffffu, ok);
    // inclusive scan of need over the k <= 16 member lanes
    int64_t incl = need;
    if (k > 1) {
#pragma unroll
        for (int o = 1; o < PL_MAXK; o <<= 1) {
            const int64_t u = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += u;
        }
    }
    if (lane < k) pl.need_off[lane + 1] = incl;
    if (lane == 0) {
        pl.need_off[0] = 0;
        pl.ok = all_ok ? 1 : 0;
    }
    __syncwarp();
}

// never_fits (scheduler.cpp:225-243): uses the first instance's capacity.
__device__ __forceinline__ bool never_fits_d(const PlannerState& st, int64_t L, int k_dcp) {
    const int64_t demand = pages_for_d(L, st.page);
    const int64_t per = st.capacity;
    int64_t reach;
    if (st.kind == KIND_DCP) {
        const int k = k_dcp;
        reach = per * k - (k - 1);
    } else if (st.kind == KIND_UNIFORM) {
        reach = per * st.udeg - (st.udeg - 1);
    } else {
        reach = per;
    }
    return demand > reach;
}

// ------------------------------------------------------------------ single-CTA bitonic sort
// Sorts n (<= sort_cap, padded to pow2 internally) entries by (k1, k2) ascending.
static __device__ void cta_bitonic_sort(int64_t* k1, int64_t* k2, int32_t* val, int n) {
    int np2 = 1;
    while (np2 < n) np2 <<= 1;
    for (int i = n + threadIdx.x; i < np2; i += blockDim.x) {
        k1[i] = INT64_MAX;
        k2[i] = INT64_MAX;
        val[i] = -1;
    }
    __syncthreads();
    for (int size = 2; size <= np2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < np2 / 2; i += blockDim.x) {
                const int lo = 2 * i - (i & (stride - 1));
                const int hi = lo + stride;
                const bool up = ((lo & size) == 0);
                const bool gt = k1[lo] > k1[hi] || (k1[lo] == k1[hi] && k2[lo] > k2[hi]);
                if (gt == up) {
                    int64_t t1 = k1[lo]; k1[lo] = k1[hi]; k1[hi] = t1;
                    int64_t t2 = k2[lo]; k2[lo] = k2[hi]; k2[hi] = t2;
                    int32_t tv = val[lo]; val[lo] = val[hi]; val[hi] = tv;
                }
            }
            __syncthreads();
        }
    }
}

// rebalance_active (scheduler.cpp:43-64) on the shared-memory B (already
// zeroed): the given slots, or every ACTIVE slot when slots == nullptr.
// (cp_degree, id) order: CP=1 first (m_r pinned, parallel histogram), then the
// CP>=2 requests sequentially with a warp argmin over P_r.
// The CP >= 2 requests (a few percent of the actives) are gathered with their kv membership
// mask into shared memory, sorted there, and assigned by warp 0 without global round trips;
// more than RB_SMEM of them fall back to the global-memory sort.
constexpr int RB_SMEM = 512;

static __device__ void rebalance_core(const PlannerState& st, SmemInst& si, int32_t& s_n2, const int32_t* slots,
                               int n) {
    __shared__ int64_t rb_id[RB_SMEM];
    __shared__ int32_t rb_k[RB_SMEM], rb_sl[RB_SMEM];
    __shared__ uint32_t rb_mask[RB_SMEM];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int S = st.max_slots;
    const int lim = slots ? n : S;
    constexpr int RU = 8;  // slots per thread per round: every dependent load level issued together
    for (int j0 = tid; j0 < lim; j0 += RU * blockDim.x) {
        int sls[RU], kks[RU], s1[RU];
#pragma unroll
        for (int u = 0; u < RU; ++u) {
            const int j = j0 + u * blockDim.x;
            sls[u] = j < lim ? (slots ? slots[j] : j) : -1;
        }
#pragma unroll
        for (int u = 0; u < RU; ++u)
            if (sls[u] >= 0 && !slots && st.state[sls[u]] != ST_ACTIVE) sls[u] = -1;
#pragma unroll
        for (int u = 0; u < RU; ++u) {
            kks[u] = sls[u] >= 0 ? st.k[sls[u]] : 0;
            s1[u] = sls[u] >= 0 ? st.kv[sls[u] * PL_MAXK] : 0;
        }
#pragma unroll
        for (int u = 0; u < RU; ++u) {
            const int sl = sls[u];
            if (sl < 0) continue;
            const int kk = kks[u];
            if (kk == 1) {
                const int s = s1[u];
                st.moe[sl] = s;
                atomicAdd(&si.B[s], 1);
            } else {
                const int i = atomicAdd(&s_n2, 1);
                st.sk1[i] = kk;
                st.sk2[i] = st.id[sl];
                st.sval[i] = sl;
                if (i < RB_SMEM) {
                    uint32_t mask = 0;
                    for (int m = 0; m < kk; ++m) mask |= 1u << st.kv[sl * PL_MAXK + m];
                    rb_k[i] = kk;
                    rb_id[i] = st.id[sl];
                    rb_sl[i] = sl;
                    rb_mask[i] = mask;
                }
            }
        }
    }
    __syncthreads();
    const int n2 = s_n2;
    if (n2 <= RB_SMEM) {
        // bitonic sort by (cp_degree, id) in shared memory
        int np2 = 1;
        while (np2 < n2) np2 <<= 1;
        for (int i = n2 + tid; i < np2; i += blockDim.x) {
            rb_k[i] = 0x7fffffff;
            rb_id[i] = INT64_MAX;
        }
        __syncthreads();
        for (int size = 2; size <= np2; size <<= 1)
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int i = tid; i < np2 / 2; i += blockDim.x) {
                    const int lo = 2 * i - (i & (stride - 1)), hi = lo + stride;
                    const bool gt = rb_k[lo] > rb_k[hi] || (rb_k[lo] == rb_k[hi] && rb_id[lo] > rb_id[hi]);
                    if (gt == ((lo & size) == 0)) {
                        const int tk = rb_k[lo]; rb_k[lo] = rb_k[hi]; rb_k[hi] = tk;
                        const int64_t ti = rb_id[lo]; rb_id[lo] = rb_id[hi]; rb_id[hi] = ti;
                        const int ts = rb_sl[lo]; rb_sl[lo] = rb_sl[hi]; rb_sl[hi] = ts;
                        const uint32_t tm = rb_mask[lo]; rb_mask[lo] = rb_mask[hi]; rb_mask[hi] = tm;
                    }
                }
                __syncthreads();
            }
        if (warp == 0) {
            for (int i = 0; i < n2; ++i) {
                // argmin over P_r of B, ties to the lowest instance id (cpp:54-59); lane = instance
                const bool mem = lane < st.W && ((rb_mask[i] >> lane) & 1u);
                const int bs = warp_argmin_small(static_cast<uint32_t>(si.B[lane]), mem, lane);
                if (lane == 0) {
                    st.moe[rb_sl[i]] = bs;
                    si.B[bs] += 1;
                }
                __syncwarp();
            }
        }
        __syncthreads();
        return;
    }
    cta_bitonic_sort(st.sk1, st.sk2, st.sval, n2);
    __syncthreads();
    if (warp == 0) {
        for (int i = 0; i < n2; ++i) {
            const int sl = st.sval[i];
            const int kk = st.k[sl];
            const int s = lane < kk ? st.kv[sl * PL_MAXK + lane] : 0;
            // argmin over P_r of B, ties to the lowest instance id (cpp:54-59): key (B_s, s)
            const int bs = warp_argmin_small(static_cast<uint32_t>(si.B[s]), lane < kk, s);
            if (lane == 0) {
                st.moe[sl] = bs;
                si.B[bs] += 1;
            }
            __syncwarp();
        }
    }
    __syncthreads();
}

// ------------------------------------------------------------------ K6 step
static __global__ void __launch_bounds__(PL_THREADS, 1) planner_step_kernel(PlannerState st) {
    __shared__ SmemInst si;
    __shared__ SmemPlace pl;
    __shared__ int32_t s_n2;
    __shared__ int32_t s_cnt[3];
    __shared__ int64_t s_hol;
    __shared__ int32_t s_status;
    __shared__ int64_t s_arena_top;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int W = st.W;
    const int S = st.max_slots;

    if (tid < W) {
        si.K[tid] = st.kv_load[tid];
        si.nfree[tid] = st.nfree[tid];
        si.B[tid] = 0;
        si.shards[tid] = st.shard_count[tid];
    }
    if (tid == 0) {
        s_n2 = 0;
        s_cnt[0] = s_cnt[1] = s_cnt[2] = 0;
        s_hol = 0;
        s_status = PL_OK;
        s_arena_top = *st.arena_top;
    }
    __syncthreads();

#ifdef DCP_PLANNER_PROF
    long long prof_t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(prof_t0));
#define PL_PROF(tag)                                                                  \
    do {                                                                              \
        long long t_;                                                                 \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                        \
        if (tid == 0) printf("planner_step %s %lld ns\n", tag, t_ - prof_t0);          \
    } while (0)
    long long plp[5] = {0, 0, 0, 0, 0}, plp_last = 0;
#define PLP_MARK(k)                                         \
    do {                                                    \
        const long long c_ = clock64();                     \
        if ((k) > 0) plp[k] += c_ - plp_last;               \
        plp_last = c_;                                      \
    } while (0)
#else
#define PL_PROF(tag) do {} while (0)
#define PLP_MARK(k) do {} while (0)
#endif
    // ---- Alg. 1 line 1: recompute B (scheduler.cpp:250-261) ----
    if (st.kind == KIND_DCP) {
        rebalance_core(st, si, s_n2, nullptr, 0);
    } else {
        for (int sl = tid; sl < S; sl += blockDim.x)
            if (st.state[sl] == ST_ACTIVE) atomicAdd(&si.B[st.moe[sl]], 1);
    }
    __syncthreads();
    PL_PROF("rebalance");

    // ---- FIFO admission (scheduler.cpp:263-304) ----
    // Warp 0 walks the queue alone (warp argmin / water_fill / can_allocate with one lane per
    // instance, no CTA barrier per request) and records each commit's frame pops; the copy of
    // the popped frame ids runs afterwards over the whole GPU (planner_pages_kernel).  The pops
    // can be deferred because admission only moves each stack's top (nfree), never its contents.
    __shared__ int32_t s_wq, s_i;
    const int nw = *st.nwait;
    if (warp == 0) {
        int wq = 0;              // entries kept so far == the reference's `scan`
        bool head_recorded = false;
        int i = 0;
        int64_t arena_top = s_arena_top;
        int64_t pbase = 0;
        int32_t q_sl = 0;        // lane j holds queue entry i0 + j (prefetched 32 at a time)
        int64_t q_len = 0;
        int i0 = -64;
        for (; i < nw; ++i) {
            if (i - i0 >= 32) {
                i0 = i;
                if (i + lane < nw) {
                    q_sl = st.waiting[i + lane];
                    q_len = st.seq_len[q_sl];
                }
            }
            PLP_MARK(0);
            const int sl = __shfl_sync(0xffffffffu, q_sl, i - i0);
            const int64_t L = __shfl_sync(0xffffffffu, q_len, i - i0);
            PLP_MARK(1);
            const int k_dcp = st.kind == KIND_DCP ? cp_degree_d(st, L) : 1;
            if (never_fits_d(st, L, k_dcp)) {  // -> unschedulable, erased
                if (lane == 0) st.res_slots[2 * S + s_cnt[2]++] = sl;
                continue;
            }
            PLP_MARK(2);
            place_request(st, si, pl, lane, L, k_dcp);
            PLP_MARK(3);
            if (pl.ok) {
                // GlobalPageTable::allocate (page_table.cpp:9-49)
                const int k = pl.k;
                const int64_t np = pl.need_off[k];
                const int64_t cap = np + st.reserve_pages;
                const int64_t off = arena_top;
                if (L < 1 || off + cap > st.arena_cap) {
                    if (lane == 0) s_status = L < 1 ? PL_E_FRAMES : PL_E_ARENA;
                    break;
                }
                PageRec& rc = st.recs[s_cnt[0]];
                if (lane < k) {  // one lane per member (members are distinct instances)
                    const int s = pl.kv[lane];
                    rc.kv[lane] = s;
                    rc.top[lane] = si.nfree[s];
                    rc.split[lane] = pl.split[lane];
                    rc.need_off[lane + 1] = pl.need_off[lane + 1];
                    si.nfree[s] -= pl.need_off[lane + 1] - pl.need_off[lane];
                    si.K[s] += pl.split[lane];
                    si.shards[s] += 1;
                }
                __syncwarp();  // every lane has read s_cnt[0] / pl before lane 0 advances them
                if (lane == 0) {
                    rc.need_off[0] = 0;
                    *reinterpret_cast<longlong2*>(&rc.base) = make_longlong2(pbase, off);
                    *reinterpret_cast<int4*>(&rc.k) = make_int4(k, sl, pl.moe, (int32_t)cap);
                    si.B[pl.moe] += 1;
                    st.res_slots[s_cnt[0]++] = sl;
                }
                arena_top = off + cap;
                pbase += np;
                __syncwarp();
                PLP_MARK(4);
                continue;
            }
            // deferred (cpp:296-303)
            const int64_t tf = warp_sum_i64(lane < W ? si.nfree[lane] : 0);
            if (lane == 0) {
                st.res_slots[S + s_cnt[1]++] = sl;
                if (wq == 0 && !head_recorded) {
                    if (tf >= pages_for_d(L, st.page)) s_hol += 1;
                }
                st.waiting[wq] = sl;
            }
            head_recorded = head_recorded || (wq == 0);
            ++wq;
            __syncwarp();  // every lane has read pl before the next placement rewrites it
            if (st.hol_strict) {
                ++i;
                break;
            }
        }
        __syncwarp();  // the lanes' initial read of s_arena_top precedes lane 0's write
        if (lane == 0) {
            s_arena_top = arena_top;
            *st.res_pages = pbase;
            s_wq = wq;
            s_i = i;
        }
    }
    __syncthreads();
    // planner_pages_kernel's CTAs may launch now.  Not earlier: its parked CTAs would share this
    // SM with the one-warp admission loop above (K6 64-admission round 110 -> 165 us when the
    // trigger sat at the kernel's entry).
    pdl_trigger();
    PL_PROF("admission");
#ifdef DCP_PLANNER_PROF
    if (tid == 0) printf("sections(cycles): prefetch %lld nf %lld place %lld commit %lld\n", plp[1], plp[2], plp[3], plp[4]);
#endif
    int wq = s_wq;
    const int i = s_i;
    // keep the untouched tail of the queue in order (wq <= i: a downward move, chunk by chunk)
    for (int c = 0; c < nw - i; c += blockDim.x) {
        const int j = i + c + tid;
        const int32_t v = j < nw ? st.waiting[j] : 0;
        __syncthreads();
        if (j < nw) st.waiting[wq + c + tid] = v;
        __syncthreads();
    }
    wq += nw - i;
    __syncthreads();
    PL_PROF("tail");
    if (tid < W) {
        st.kv_load[tid] = si.K[tid];
        st.nfree[tid] = si.nfree[tid];
        st.moe_batch[tid] = si.B[tid];
        st.shard_count[tid] = si.shards[tid];
    }
    if (tid == 0) {
        *st.nwait = wq;
        *st.arena_top = s_arena_top;
        st.res_counts[0] = s_cnt[0];
        st.res_counts[1] = s_cnt[1];
        st.res_counts[2] = s_cnt[2];
        st.res_counts[3] = s_status;
        *st.res_hol = s_hol;
    }
}

// The frame pops of the step's commits (page_table.cpp:30-45): page g of the step's commit
// list -> (commit, member, page j of that member) -> the member's stack entry top - 1 - j.
// Grid-stride over every page the step popped, UP pages per thread per round, loads first.
static __global__ void __launch_bounds__(256) planner_pages_kernel(PlannerState st) {
    pdl_wait();  // PDL-launched after planner_step_kernel (its commit records)
    const int64_t ptot = *st.res_pages;
    const int nrec = st.res_counts[0];
    // the commits' slot fields (allocate(), page_table.cpp:9-49; Request::placement / state)
    for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < nrec; c += gridDim.x * blockDim.x) {
        const PageRec& rc = st.recs[c];
        const int sl = rc.sl, k = rc.k;
        int64_t trailing = 0;
        for (int m = 0; m < k; ++m) {
            st.kv[sl * PL_MAXK + m] = rc.kv[m];
            st.split[sl * PL_MAXK + m] = rc.split[m];
            if (rc.split[m] > 0) {  // the last member with tokens holds the trailing page
                const int64_t r = page_rem_d(rc.split[m], st.page);
                trailing = r == 0 ? st.page : r;
            }
        }
        for (int s = 0; s < st.W; ++s) {
            int64_t v = 0;
            for (int m = 0; m < k; ++m)
                if (rc.kv[m] == s) v = rc.split[m];
            st.shard_tokens[(int64_t)sl * st.W + s] = v;
        }
        st.k[sl] = k;
        st.moe[sl] = rc.moe;
        st.state[sl] = ST_ACTIVE;
        st.page_off[sl] = rc.off;
        st.page_cnt[sl] = (int32_t)rc.need_off[k];
        st.page_cap[sl] = rc.cap;
        st.trailing_fill[sl] = trailing;
    }
    constexpr int UP = 4;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t g0 = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; g0 < ptot; g0 += UP * stride) {
        int32_t fr[UP];
        int rs[UP], ms[UP];
#pragma unroll
        for (int u = 0; u < UP; ++u) {
            const int64_t g = g0 + u * stride;
            int r = 0, m = 0;
            if (g < ptot) {
                int hi = nrec - 1;  // last commit with base <= g
                while (r < hi) {
                    const int mid = (r + hi + 1) >> 1;
                    if (st.recs[mid].base <= g) r = mid; else hi = mid - 1;
                }
                const PageRec& rc = st.recs[r];
                const int64_t t = g - rc.base;
                while (rc.need_off[m + 1] <= t) ++m;
                fr[u] = st.stack[(int64_t)rc.kv[m] * st.capacity + rc.top[m] - 1 - (t - rc.need_off[m])];
            }
            rs[u] = r;
            ms[u] = m;
        }
#pragma unroll
        for (int u = 0; u < UP; ++u) {
            const int64_t g = g0 + u * stride;
            if (g >= ptot) break;
            const PageRec& rc = st.recs[rs[u]];
            const int m = ms[u];
            const int64_t t = g - rc.base;
            const int64_t j = t - rc.need_off[m];
            st.pg_inst[rc.off + t] = rc.kv[m];
            st.pg_frame[rc.off + t] = fr[u];
            const int64_t rem = rc.split[m] - j * st.page;
            st.pg_fill[rc.off + t] = (uint8_t)(rem < st.page ? rem : st.page);
        }
    }
}

// ------------------------------------------------------------------ release (pt_free)
// GlobalPageTable::release (page_table.cpp:51-66): frames pushed back in page
// order, K_s -= shard tokens.  Requests are released sequentially in the given
// order (the LIFO contents depend on it); each request's pages are pushed in
// parallel with per-instance stable ranks.
static __global__ void __launch_bounds__(PL_THREADS, 1)
    planner_release_kernel(PlannerState st, const int32_t* slots, int n) {
    __shared__ int32_t cnt[PL_THREADS / 32][PL_MAXW];
    __shared__ int64_t base[PL_MAXW];
    __shared__ int64_t nfree[PL_MAXW];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int W = st.W;
    constexpr int NWARP = PL_THREADS / 32;
    if (tid < W) nfree[tid] = st.nfree[tid];
    __syncthreads();
    for (int q = 0; q < n; ++q) {
        const int sl = slots[q];
        const int64_t off = st.page_off[sl];
        const int np = st.page_cnt[sl];
        for (int c0 = 0; c0 < np; c0 += PL_THREADS) {
            const int t = c0 + tid;
            const bool live = t < np;
            const int s = live ? st.pg_inst[off + t] : -1;
            const unsigned same = __match_any_sync(0xffffffffu, s);
            const int rank = __popc(same & ((1u << lane) - 1u));
            for (int j = lane; j < W; j += 32) cnt[warp][j] = 0;
            __syncwarp();
            if (live && rank == 0) cnt[warp][s] = __popc(same);
            __syncthreads();
            if (tid < W) {  // exclusive scan over warps per instance
                int64_t run = 0;
                for (int w = 0; w < NWARP; ++w) {
                    const int c = cnt[w][tid];
                    cnt[w][tid] = (int32_t)run;
                    run += c;
                }
                base[tid] = run;  // total in this chunk
            }
            __syncthreads();
            if (live) {
                const int64_t pos = nfree[s] + cnt[warp][s] + rank;
                st.stack[(int64_t)s * st.capacity + pos] = st.pg_frame[off + t];
            }
            __syncthreads();
            if (tid < W) nfree[tid] += base[tid];
            __syncthreads();
        }
        if (tid < W) st.kv_load[tid] -= st.shard_tokens[(int64_t)sl * W + tid];
        if (tid == 0) st.state[sl] = ST_FINISHED;
        __syncthreads();
    }
    if (tid < W) st.nfree[tid] = nfree[tid];
}

// ------------------------------------------------------------------ append_token
// GlobalPageTable::append_token (page_table.cpp:86-121), sequential over the
// batch (frames popped depend on order).  out_inst[q] = receiving instance or
// -1 (growth stall).  Stops with PL_E_ARENA at the first request whose page
// segment must grow past the arena; res_counts[0] = processed count.
static __global__ void planner_append_kernel(PlannerState st, const int32_t* slots, int n,
                                      int32_t* out_inst) {
    const int lane = threadIdx.x & 31;
    const int W = st.W;
    int q = 0;
    int status = PL_OK;
    for (; q < n; ++q) {
        const int sl = slots[q];
        int64_t off = st.page_off[sl];
        const int cnt = st.page_cnt[sl];
        int target;
        if (cnt > 0 && st.trailing_fill[sl] < st.page) {
            target = st.pg_inst[off + cnt - 1];
            if (lane == 0) {
                st.trailing_fill[sl] += 1;
                st.pg_fill[off + cnt - 1] += 1;
                st.kv_load[target] += 1;
                st.shard_tokens[(int64_t)sl * W + target] += 1;
                st.generated[sl] += 1;
                st.last_append[sl] = target;
                out_inst[q] = target;
            }
            __syncwarp();
            continue;
        }
        target = cnt == 0 ? st.kv[sl * PL_MAXK] : st.pg_inst[off + cnt - 1];
        if (st.nfree[target] == 0) {
            target = -1;
            for (int m = 0; m < st.k[sl]; ++m) {
                const int s = st.kv[sl * PL_MAXK + m];
                if (st.nfree[s] > 0) { target = s; break; }
            }
        }
        if (target < 0) {
            if (lane == 0) {
                out_inst[q] = -1;
                st.last_append[sl] = -1;
            }
            __syncwarp();
            continue;
        }
        if (cnt == st.page_cap[sl]) {  // grow the page segment (vector-style)
            const int newcap = cnt * 2 > cnt + 16 ? cnt * 2 : cnt + 16;
            const int64_t noff = *st.arena_top;
            if (noff + newcap > st.arena_cap) {
                status = PL_E_ARENA;
                break;
            }
            for (int t = lane; t < cnt; t += 32) {
                st.pg_inst[noff + t] = st.pg_inst[off + t];
                st.pg_frame[noff + t] = st.pg_frame[off + t];
                st.pg_fill[noff + t] = st.pg_fill[off + t];
            }
            __syncwarp();
            if (lane == 0) {
                *st.arena_top = noff + newcap;
                st.page_off[sl] = noff;
                st.page_cap[sl] = newcap;
            }
            __syncwarp();
            off = noff;
        }
        if (lane == 0) {
            const int64_t nf = st.nfree[target];
            st.pg_inst[off + cnt] = target;
            st.pg_frame[off + cnt] = st.stack[(int64_t)target * st.capacity + nf - 1];
            st.pg_fill[off + cnt] = 1;
            st.nfree[target] = nf - 1;
            st.page_cnt[sl] = cnt + 1;
            st.trailing_fill[sl] = 1;
            st.kv_load[target] += 1;
            st.shard_tokens[(int64_t)sl * W + target] += 1;
            st.generated[sl] += 1;
            st.last_append[sl] = target;
            out_inst[q] = target;
        }
        __syncwarp();
    }
    if (lane == 0) {
        st.res_counts[0] = q;
        st.res_counts[3] = status;
    }
}


// ------------------------------------------------------------------ append_token, batched
// The same semantics as planner_append_kernel for a batch WITHOUT duplicate
// requests, in parallel: a request appends to its trailing page when it has
// room; otherwise it takes the top free frame of the instance holding its last
// page.  Requests needing a frame on the same instance pop consecutive stack
// entries in batch order (per-instance ranks from a block scan), which is what
// the sequential loop does as long as no instance runs out.  When some
// instance's demand exceeds its free frames (the fallback path of
// page_table.cpp:104-113 would trigger) or the page arena cannot absorb the
// segment growth, nothing is mutated and res_counts[2] = 1 asks the host to
// run the sequential kernel instead.
constexpr int PL_APPEND_THREADS = 256;
static __global__ void __launch_bounds__(PL_APPEND_THREADS, 1)
    planner_append_parallel_kernel(PlannerState st, const int32_t* slots, int n, int32_t* out_inst) {
    __shared__ int32_t cnt[PL_APPEND_THREADS][PL_MAXW];
    __shared__ int64_t grow_part[PL_APPEND_THREADS];
    __shared__ int32_t demand[PL_MAXW];
    __shared__ int32_t bail;
    __shared__ unsigned long long kv_add[PL_MAXW];
    __shared__ int64_t arena_base;
    const int tid = threadIdx.x, W = st.W;
    const int per = (n + blockDim.x - 1) / blockDim.x;
    const int q0 = min(n, tid * per), q1 = min(n, (tid + 1) * per);
    for (int s = 0; s < W; ++s) cnt[tid][s] = 0;
    int64_t grow = 0;
    for (int q = q0; q < q1; ++q) {
        const int sl = slots[q];
        const int c = st.page_cnt[sl];
        if (c > 0 && st.trailing_fill[sl] < st.page) continue;
        const int tgt = c == 0 ? st.kv[sl * PL_MAXK] : st.pg_inst[st.page_off[sl] + c - 1];
        cnt[tid][tgt] += 1;
        if (c == st.page_cap[sl]) grow += c * 2 > c + 16 ? c * 2 : c + 16;
    }
    grow_part[tid] = grow;
    if (tid < W) kv_add[tid] = 0;
    __syncthreads();
    if (tid < W) {  // exclusive scan over threads per instance
        int run = 0;
        for (int t = 0; t < (int)blockDim.x; ++t) {
            const int v = cnt[t][tid];
            cnt[t][tid] = run;
            run += v;
        }
        demand[tid] = run;
    }
    if (tid == 0) {
        int64_t g = 0;
        for (int t = 0; t < (int)blockDim.x; ++t) {
            const int64_t v = grow_part[t];
            grow_part[t] = g;
            g += v;
        }
        bail = (*st.arena_top + g > st.arena_cap) ? 1 : 0;
        arena_base = *st.arena_top;
        if (!bail) *st.arena_top = arena_base + g;
    }
    __syncthreads();
    if (tid < W && demand[tid] > st.nfree[tid]) atomicExch(&bail, 1);
    __syncthreads();
    if (bail) {
        if (tid == 0) {
            if (arena_base != *st.arena_top) *st.arena_top = arena_base;
            st.res_counts[0] = 0;
            st.res_counts[2] = 1;
            st.res_counts[3] = PL_OK;
        }
        return;
    }
    int rank[PL_MAXW];
    for (int s = 0; s < W; ++s) rank[s] = cnt[tid][s];
    int64_t goff = arena_base + grow_part[tid];
    for (int q = q0; q < q1; ++q) {
        const int sl = slots[q];
        int64_t off = st.page_off[sl];
        const int c = st.page_cnt[sl];
        int tgt;
        if (c > 0 && st.trailing_fill[sl] < st.page) {
            tgt = st.pg_inst[off + c - 1];
            st.trailing_fill[sl] += 1;
            st.pg_fill[off + c - 1] += 1;
        } else {
            tgt = c == 0 ? st.kv[sl * PL_MAXK] : st.pg_inst[off + c - 1];
            if (c == st.page_cap[sl]) {
                const int newcap = c * 2 > c + 16 ? c * 2 : c + 16;
                for (int t = 0; t < c; ++t) {
                    st.pg_inst[goff + t] = st.pg_inst[off + t];
                    st.pg_frame[goff + t] = st.pg_frame[off + t];
                    st.pg_fill[goff + t] = st.pg_fill[off + t];
                }
                st.page_off[sl] = goff;
                st.page_cap[sl] = newcap;
                off = goff;
                goff += newcap;
            }
            const int64_t pos = st.nfree[tgt] - 1 - rank[tgt];
            rank[tgt] += 1;
            st.pg_inst[off + c] = tgt;
            st.pg_frame[off + c] = st.stack[(int64_t)tgt * st.capacity + pos];
            st.pg_fill[off + c] = 1;
            st.page_cnt[sl] = c + 1;
            st.trailing_fill[sl] = 1;
        }
        atomicAdd(&kv_add[tgt], 1ull);
        st.shard_tokens[(int64_t)sl * W + tgt] += 1;
        st.generated[sl] += 1;
        st.last_append[sl] = tgt;
        out_inst[q] = tgt;
    }
    __syncthreads();
    if (tid < W) {
        st.nfree[tid] -= demand[tid];
        st.kv_load[tid] += (int64_t)kv_add[tid];
    }
    if (tid == 0) {
        st.res_counts[0] = n;
        st.res_counts[2] = 0;
        st.res_counts[3] = PL_OK;
    }
}

// ------------------------------------------------------------------ arena compaction
// Moves every live page segment (ACTIVE slots) to a fresh arena, packed in slot order.
static __global__ void planner_compact_offsets(PlannerState st, int64_t* new_off) {
    __shared__ int64_t part[1024];
    const int tid = threadIdx.x;
    const int S = st.max_slots;
    const int per = (S + blockDim.x - 1) / blockDim.x;
    int64_t sum = 0;
    for (int j = tid * per; j < min(S, (tid + 1) * per); ++j)
        if (st.state[j] == ST_ACTIVE) sum += st.page_cap[j];
    part[tid] = sum;
    __syncthreads();
    if (tid == 0) {
        int64_t run = 0;
        for (int t = 0; t < (int)blockDim.x; ++t) {
            const int64_t v = part[t];
            part[t] = run;
            run += v;
        }
        *st.arena_top = run;
    }
    __syncthreads();
    int64_t run = part[tid];
    for (int j = tid * per; j < min(S, (tid + 1) * per); ++j) {
        new_off[j] = run;
        if (st.state[j] == ST_ACTIVE) run += st.page_cap[j];
    }
}

static __global__ void planner_compact_copy(PlannerState st, const int64_t* new_off, int32_t* inst2,
                                     int32_t* frame2, uint8_t* fill2) {
    const int sl = blockIdx.x;
    if (st.state[sl] != ST_ACTIVE) return;
    const int64_t off = st.page_off[sl], noff = new_off[sl];
    for (int t = threadIdx.x; t < st.page_cnt[sl]; t += blockDim.x) {
        inst2[noff + t] = st.pg_inst[off + t];
        frame2[noff + t] = st.pg_frame[off + t];
        fill2[noff + t] = st.pg_fill[off + t];
    }
    __syncthreads();
    if (threadIdx.x == 0) st.page_off[sl] = noff;
}


// ------------------------------------------------------------------ standalone entry kernels
// rebalance_active over an explicit active list (scheduler.cpp:43-64): B is
// reset for every instance, then recomputed from the list only.
static __global__ void __launch_bounds__(PL_THREADS, 1)
    planner_rebalance_kernel(PlannerState st, const int32_t* slots, int n) {
    __shared__ SmemInst si;
    __shared__ int32_t s_n2;
    if (threadIdx.x < st.W) si.B[threadIdx.x] = 0;
    if (threadIdx.x == 0) s_n2 = 0;
    __syncthreads();
    rebalance_core(st, si, s_n2, slots, n);
    if (threadIdx.x < st.W) st.moe_batch[threadIdx.x] = si.B[threadIdx.x];
}

// GlobalPageTable::allocate with a caller-supplied placement (page_table.cpp:9-49):
// feasibility first (no partial state on failure), then LIFO pops in
// kv_binding order.  Does not touch B_s / R_i (those belong to Scheduler::step).
static __global__ void __launch_bounds__(PL_THREADS, 1)
    planner_allocate_kernel(PlannerState st, int sl, int k, const int32_t* kv, const int64_t* split, int moe) {
    __shared__ int64_t need_off[PL_MAXK + 1];
    __shared__ int32_t ok;
    const int tid = threadIdx.x;
    if (tid == 0) {
        need_off[0] = 0;
        ok = st.seq_len[sl] >= 1;
        for (int m = 0; m < k; ++m) {
            const int64_t need = pages_for_d(split[m], st.page);
            if (st.nfree[kv[m]] < need) ok = 0;
            need_off[m + 1] = need_off[m] + need;
        }
        if (*st.arena_top + need_off[k] + st.reserve_pages > st.arena_cap) ok = -1;
    }
    __syncthreads();
    if (ok != 1) {
        if (tid == 0) st.res_counts[3] = ok == 0 ? PL_E_FRAMES : PL_E_ARENA;
        return;
    }
    const int64_t np = need_off[k];
    const int64_t off = *st.arena_top;
    for (int64_t t = tid; t < np; t += blockDim.x) {
        int m = 0;
        while (need_off[m + 1] <= t) ++m;
        const int s = kv[m];
        const int64_t j = t - need_off[m];
        st.pg_inst[off + t] = s;
        st.pg_frame[off + t] = st.stack[(int64_t)s * st.capacity + st.nfree[s] - 1 - j];
        const int64_t rem = split[m] - j * st.page;
        st.pg_fill[off + t] = (uint8_t)(rem < st.page ? rem : st.page);
    }
    __syncthreads();
    if (tid == 0) {
        const int W = st.W;
        for (int s = 0; s < W; ++s) st.shard_tokens[(int64_t)sl * W + s] = 0;
        int64_t trailing = 0;
        for (int m = 0; m < k; ++m) {
            const int s = kv[m];
            st.nfree[s] -= need_off[m + 1] - need_off[m];
            st.kv_load[s] += split[m];
            st.shard_tokens[(int64_t)sl * W + s] += split[m];
            st.kv[sl * PL_MAXK + m] = s;
            st.split[sl * PL_MAXK + m] = split[m];
            if (split[m] > 0) {
                const int64_t r = page_rem_d(split[m], st.page);
                trailing = r == 0 ? st.page : r;
            }
        }
        st.k[sl] = k;
        st.moe[sl] = moe;
        st.state[sl] = ST_ACTIVE;
        st.page_off[sl] = off;
        st.page_cnt[sl] = (int32_t)np;
        st.page_cap[sl] = (int32_t)(np + st.reserve_pages);
        st.trailing_fill[sl] = trailing;
        *st.arena_top = off + np + st.reserve_pages;
        st.res_counts[3] = PL_OK;
    }
}

// water_fill (scheduler.cpp:70-102) for one participant list, one warp.
static __global__ void water_fill_kernel(int n, const int64_t* loads, int64_t len, int64_t* split) {
    const int lane = threadIdx.x & 31;
    const int64_t K = lane < n ? loads[lane] : 0;
    const int64_t s = warp_water_fill(lane, n, len, K);
    if (lane < n) split[lane] = s;
}

}  // namespace dcp
