// SPDX-License-Identifier: Apache-2.0
//
// K7: lowering of committed placements to per-instance metadata (north_star
// subsystem 4), restating bit-exactly
//   build_binding_config   routing.cpp:9-32   (M / N lists ordered by request id,
//                                             zero-split members included)
//   derive_routing_tables  routing.cpp:34-63  (q_route N x W one-hot at m_r,
//                                             res_route M x W ones at P_r)
//   bucket_shape           routing.cpp:89-109 (default 48-bucket space)
// and additionally emitting each instance's K1 inputs (the shard list = the N
// list, its block table, per-page fill and shard lengths) so the planner's
// output feeds the attention kernel without leaving the device.
//
// r1 (1 CTA x 32 warps): sort ACTIVE slots by id, then warp s builds instance
// s's M/N rows with ballots (stable, id order).  r2 (1 CTA per instance):
// count each row's pages on the instance, block-scan, scatter frames in
// logical page order.
#pragma once

#include <cstdint>

#include "planner.cuh"
#include "ptx.cuh"

namespace dcp {

struct RoutingOut {
    int32_t* n_count;     // [W]
    int32_t* m_count;     // [W]
    int64_t* n_id;        // [W][S]
    int32_t* n_slot;      // [W][S]
    int32_t* n_moe;       // [W][S]  shard_request_moe
    uint8_t* q_route;     // [W][S][W]
    int64_t* m_id;        // [W][S]
    int32_t* m_slot;      // [W][S]
    uint8_t* res_route;   // [W][S][W]
    int32_t* bucket;      // [W][2]  (M^, N^) or (-1,-1) on ShapeOverflow
    int32_t* cu_pages;    // [W][S+1]
    int64_t* shard_len;   // [W][S]
    int32_t* block_table; // [W][capacity]
    uint8_t* page_fill;   // [W][capacity]
    int32_t* status;      // [1]
    int32_t* n_active;    // [1] actives compacted by routing_collect_kernel
    // exchange maps (K2/K3 destinations)
    int32_t* slot_nrow;   // [S][W] row of a slot in instance s's N list
    int32_t* slot_mrow;   // [S]    row of a slot in m_r's M list
    int32_t* n_mrow;      // [W][S] for N row: row in m_r's M list
    int32_t* m_nrow;      // [W][S][W] for M row: row in s' N list, -1 if s' not in P_r
    int32_t* m_k;         // [W][S] |P_r|
    int32_t* m_kv;        // [W][S][PL_MAXK] P_r in kv_binding order
};

__device__ __forceinline__ void bucket_shape_default_d(int m, int n, int32_t* out) {
    const int ms[6] = {8, 16, 32, 64, 128, 256};
    const int ns[8] = {8, 16, 32, 64, 128, 256, 384, 512};
    if (m > 256 || n > 512) {
        out[0] = out[1] = -1;  // ShapeOverflow (routing.cpp:102-105)
        return;
    }
    for (int i = 0; i < 6; ++i)
        for (int j = 0; j < 8; ++j)
            if (ms[i] >= m && ns[j] >= n) {
                out[0] = ms[i];
                out[1] = ns[j];
                return;
            }
    out[0] = 256;
    out[1] = 512;
}

static __global__ void __launch_bounds__(1024, 1) routing_rows_kernel(PlannerState st, RoutingOut ro) {
    pdl_trigger();  // K7 launches are PDL-chained (launch_routing_rows / dcp_planner_build_routing)
    pdl_wait();
    __shared__ int32_t s_n;
    __shared__ int32_t s_bad;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int S = st.max_slots, W = st.W;
    if (tid == 0) {
        s_n = 0;
        s_bad = 0;
    }
    __syncthreads();
    for (int sl = tid; sl < S; sl += blockDim.x) {
        if (st.state[sl] != ST_ACTIVE) continue;
        const int i = atomicAdd(&s_n, 1);
        st.sk1[i] = st.id[sl];
        st.sk2[i] = 0;
        st.sval[i] = sl;
        bool holds = false;  // InconsistentPlacement check (routing.cpp:19-21)
        for (int m = 0; m < st.k[sl]; ++m) holds |= st.kv[sl * PL_MAXK + m] == st.moe[sl];
        if (!holds) s_bad = 1;
    }
    __syncthreads();
    const int n = s_n;
    if (n > 1) cta_bitonic_sort(st.sk1, st.sk2, st.sval, n);
    __syncthreads();
    if (s_bad) {
        if (tid == 0) *ro.status = -4;
        return;
    }
    if (warp < W) {
        const int s = warp;
        int nrow = 0, mrow = 0;
        for (int c = 0; c < n; c += 32) {
            const int a = c + lane;
            bool inN = false, inM = false;
            int sl = -1;
            if (a < n) {
                sl = st.sval[a];
                for (int m = 0; m < st.k[sl]; ++m) inN |= st.kv[sl * PL_MAXK + m] == s;
                inM = st.moe[sl] == s;
            }
            const unsigned bn = __ballot_sync(0xffffffffu, inN);
            const unsigned bm = __ballot_sync(0xffffffffu, inM);
            const unsigned lt = (1u << lane) - 1u;
            if (inN) {
                const int row = nrow + __popc(bn & lt);
                const size_t r = (size_t)s * S + row;
                ro.n_id[r] = st.id[sl];
                ro.n_slot[r] = sl;
                ro.n_moe[r] = st.moe[sl];
                uint8_t* q = ro.q_route + r * W;
                for (int c2 = 0; c2 < W; ++c2) q[c2] = (c2 == st.moe[sl]) ? 1 : 0;
                ro.shard_len[r] = st.shard_tokens[(size_t)sl * W + s];
                ro.slot_nrow[(size_t)sl * W + s] = row;
            }
            if (inM) {
                const int row = mrow + __popc(bm & lt);
                const size_t r = (size_t)s * S + row;
                ro.m_id[r] = st.id[sl];
                ro.m_slot[r] = sl;
                uint8_t* q = ro.res_route + r * W;
                for (int c2 = 0; c2 < W; ++c2) q[c2] = 0;
                for (int m = 0; m < st.k[sl]; ++m) q[st.kv[sl * PL_MAXK + m]] = 1;
                ro.slot_mrow[sl] = row;
            }
            nrow += __popc(bn);
            mrow += __popc(bm);
        }
        if (lane == 0) {
            ro.n_count[s] = nrow;
            ro.m_count[s] = mrow;
            bucket_shape_default_d(mrow, nrow, ro.bucket + 2 * s);
        }
    }
    if (tid == 0) *ro.status = 0;
}

// routing_rows_kernel with the sort and the per-active data in shared memory (the common
// case: max_slots <= ROWS_SMEM_MAX).  The global-memory sort above does ~80 barrier-separated
// passes over HBM; here each pass is a few hundred cycles, and the W row-building warps scan
// (kv membership mask, moe) from shared memory instead of chasing st.k / st.kv per request.
constexpr int ROWS_SMEM_MAX = 8192;
constexpr size_t rows_smem_bytes(int np2) { return (size_t)np2 * (8 + 4 + 4 + 4); }

// One uint8 route row (RouteTable, routing.hpp:27-40): byte c = bit c of `mask`.  Rows are
// W bytes at r * W, so for W % 4 == 0 they go out as 32-bit words (4 bytes per store).
__device__ __forceinline__ void store_route_row(uint8_t* row, int W, uint32_t mask) {
    if ((W & 3) == 0) {
        for (int c = 0; c < W; c += 4) {
            const uint32_t b = mask >> c;
            reinterpret_cast<uint32_t*>(row)[c >> 2] =
                (b & 1u) | ((b >> 1) & 1u) << 8 | ((b >> 2) & 1u) << 16 | ((b >> 3) & 1u) << 24;
        }
    } else {
        for (int c = 0; c < W; ++c) row[c] = (mask >> c) & 1u;
    }
}

// Row order = request id order (build_binding_config sorts by id, routing.cpp:9-32).  The ids
// are ranked on the whole GPU instead of sorted in one CTA: routing_collect_kernel compacts the
// active slots (id -> sk2, slot -> sval, rank sk1 = 0), routing_rank_kernel counts for every
// active how many ids are smaller (equal ids, which the planner never has, rank by collection
// order), split over RK_SPLIT CTAs per 256 actives,
// and the rows kernel scatters each active to its rank.  (A one-CTA bitonic sort of 4,096
// keys took ~35 us, issue-bound on that one SM.)
constexpr int RK_SPLIT = 8;

static __global__ void __launch_bounds__(1024) routing_collect_kernel(PlannerState st, RoutingOut ro) {
    pdl_trigger();  // K7 launches are PDL-chained (launch_routing_rows / dcp_planner_build_routing)
    pdl_wait();
    __shared__ int32_t s_n;
    if (threadIdx.x == 0) s_n = 0;
    __syncthreads();
    for (int sl = threadIdx.x; sl < st.max_slots; sl += blockDim.x) {
        if (st.state[sl] != ST_ACTIVE) continue;
        const int i = atomicAdd(&s_n, 1);
        st.sk2[i] = st.id[sl];
        st.sval[i] = sl;
        st.sk1[i] = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) *ro.n_active = s_n;
}

static __global__ void __launch_bounds__(256) routing_rank_kernel(PlannerState st, RoutingOut ro) {
    pdl_trigger();  // K7 launches are PDL-chained (launch_routing_rows / dcp_planner_build_routing)
    pdl_wait();
    __shared__ int64_t tile[256];
    const int n = *ro.n_active;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (static_cast<int>(blockIdx.x * blockDim.x) >= n) return;
    const int64_t ki = i < n ? st.sk2[i] : 0;
    const int j0 = static_cast<int>(static_cast<int64_t>(blockIdx.y) * n / gridDim.y);
    const int j1 = static_cast<int>(static_cast<int64_t>(blockIdx.y + 1) * n / gridDim.y);
    unsigned long long cnt = 0;
    for (int t = j0; t < j1; t += blockDim.x) {
        const int j = t + threadIdx.x;
        tile[threadIdx.x] = j < j1 ? st.sk2[j] : INT64_MAX;
        __syncthreads();
        const int m = min(static_cast<int>(blockDim.x), j1 - t);
        for (int u = 0; u < m; ++u) cnt += tile[u] < ki || (tile[u] == ki && t + u < i);  // ties: a permutation
        __syncthreads();
    }
    if (i < n && cnt) atomicAdd(reinterpret_cast<unsigned long long*>(st.sk1 + i), cnt);
}

static __global__ void __launch_bounds__(1024, 1) routing_rows_smem_kernel(PlannerState st, RoutingOut ro, int np2cap) {
    pdl_trigger();  // K7 launches are PDL-chained (launch_routing_rows / dcp_planner_build_routing)
    pdl_wait();
#ifdef DCP_PLANNER_PROF
    long long rt_ts[6];
    int rt_n = 0;
#define RT_STAMP()                                                   \
    do {                                                             \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(rt_ts[rt_n])); \
        ++rt_n;                                                      \
    } while (0)
    RT_STAMP();
#else
#define RT_STAMP() do {} while (0)
#endif
    extern __shared__ __align__(16) uint8_t rsm[];
    int64_t* key = reinterpret_cast<int64_t*>(rsm);
    int32_t* val = reinterpret_cast<int32_t*>(key + np2cap);
    uint32_t* kvm = reinterpret_cast<uint32_t*>(val + np2cap);
    int32_t* moe = reinterpret_cast<int32_t*>(kvm + np2cap);
    __shared__ int32_t s_bad;
    const int tid = threadIdx.x;
    if (tid == 0) s_bad = 0;
    __syncthreads();
    // actives in id order: each to its rank (routing_rank_kernel)
    const int n = *ro.n_active;
    for (int i = tid; i < n; i += blockDim.x) {
        const int r = static_cast<int>(st.sk1[i]);
        key[r] = st.sk2[i];
        val[r] = st.sval[i];
    }
    __syncthreads();
    RT_STAMP();
    RT_STAMP();  // (was: the one-CTA sort)
    for (int a = tid; a < n; a += blockDim.x) {
        const int sl = val[a];
        const int k = st.k[sl], m_r = st.moe[sl];
        uint32_t mask = 0;
        bool holds = false;  // InconsistentPlacement check (routing.cpp:19-21)
        for (int m = 0; m < k; ++m) {
            const int sp = st.kv[sl * PL_MAXK + m];
            mask |= 1u << sp;
            holds |= sp == m_r;
        }
        kvm[a] = mask;
        moe[a] = m_r;
        if (!holds) s_bad = 1;
    }
    __syncthreads();
    if (s_bad) {
        if (tid == 0) *ro.status = -4;
        return;
    }
    // the id-ordered actives for routing_write_kernel: id -> sk2, slot -> sval, (P_r mask, m_r) -> sk1
    for (int a = tid; a < n; a += blockDim.x) {
        st.sk2[a] = key[a];
        st.sval[a] = val[a];
        st.sk1[a] = static_cast<int64_t>((static_cast<uint64_t>(kvm[a]) << 32) | static_cast<uint32_t>(moe[a]));
    }
#ifdef DCP_PLANNER_PROF
    __syncthreads();
    RT_STAMP();
    RT_STAMP();
    RT_STAMP();
    if (tid == 0)
        printf("routing_rows us: rank-scatter %.1f kvm %.1f\n", (rt_ts[1] - rt_ts[0]) / 1e3, (rt_ts[3] - rt_ts[2]) / 1e3);
#endif
    if (tid == 0) *ro.status = 0;
}

// M / N rows of instance blockIdx.x (build_binding_config + derive_routing_tables,
// routing.cpp:9-63): 32 warps split the id-ordered actives; pass 1 counts each warp's N / M
// members, pass 2 writes them after the counts of the lower warps.
static __global__ void __launch_bounds__(1024) routing_write_kernel(PlannerState st, RoutingOut ro) {
    pdl_trigger();  // K7 launches are PDL-chained (launch_routing_rows / dcp_planner_build_routing)
    pdl_wait();
    __shared__ int32_t seg_n[32], seg_m[32];
    if (*ro.status != 0) return;
    const int s = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int S = st.max_slots, W = st.W;
    const int n = *ro.n_active;
    const int nw = blockDim.x >> 5;
    const int a0 = (int)((int64_t)warp * n / nw), a1 = (int)((int64_t)(warp + 1) * n / nw);
    auto kvm_of = [&](int a) { return static_cast<uint32_t>(static_cast<uint64_t>(st.sk1[a]) >> 32); };
    auto moe_of = [&](int a) { return static_cast<int>(static_cast<uint32_t>(st.sk1[a])); };
    int cn = 0, cm = 0;
    for (int c = a0; c < a1; c += 32) {
        const int a = c + lane;
        const bool ok = a < a1;
        const int64_t pk = ok ? st.sk1[a] : 0;
        cn += __popc(__ballot_sync(0xffffffffu, ok && ((static_cast<uint64_t>(pk) >> (32 + s)) & 1u)));
        cm += __popc(__ballot_sync(0xffffffffu, ok && static_cast<int>(static_cast<uint32_t>(pk)) == s));
    }
    if (lane == 0) {
        seg_n[warp] = cn;
        seg_m[warp] = cm;
    }
    __syncthreads();
    int nrow = 0, mrow = 0;
    for (int j = 0; j < warp; ++j) {
        nrow += seg_n[j];
        mrow += seg_m[j];
    }
    for (int c = a0; c < a1; c += 32) {
        const int a = c + lane;
        const bool ok = a < a1;
        const uint32_t km = ok ? kvm_of(a) : 0u;
        const int mo = ok ? moe_of(a) : -1;
        const bool inN = ok && ((km >> s) & 1u);
        const bool inM = ok && mo == s;
        const int sl = ok ? st.sval[a] : 0;
        const unsigned bn = __ballot_sync(0xffffffffu, inN);
        const unsigned bm = __ballot_sync(0xffffffffu, inM);
        const unsigned lt = (1u << lane) - 1u;
        if (inN) {
            const int row = nrow + __popc(bn & lt);
            const size_t r = (size_t)s * S + row;
            ro.n_id[r] = st.sk2[a];
            ro.n_slot[r] = sl;
            ro.n_moe[r] = mo;
            store_route_row(ro.q_route + r * W, W, 1u << mo);
            ro.shard_len[r] = st.shard_tokens[(size_t)sl * W + s];
            ro.slot_nrow[(size_t)sl * W + s] = row;
        }
        if (inM) {
            const int row = mrow + __popc(bm & lt);
            const size_t r = (size_t)s * S + row;
            ro.m_id[r] = st.sk2[a];
            ro.m_slot[r] = sl;
            store_route_row(ro.res_route + r * W, W, km);
            ro.slot_mrow[sl] = row;
        }
        nrow += __popc(bn);
        mrow += __popc(bm);
    }
    if (lane == 0 && warp == nw - 1) {
        ro.n_count[s] = nrow;
        ro.m_count[s] = mrow;
        bucket_shape_default_d(mrow, nrow, ro.bucket + 2 * s);
    }
}

// Host: routing rows for the planner's active set, shared-memory sort when it fits.
static inline cudaError_t launch_routing_rows(const PlannerState& st, const RoutingOut& ro, cudaStream_t stream) {
    int np2 = 1;
    while (np2 < st.max_slots) np2 <<= 1;
    if (np2 <= ROWS_SMEM_MAX) {
        const size_t sm = rows_smem_bytes(np2);
        cudaError_t e = cudaFuncSetAttribute(routing_rows_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             static_cast<int>(sm));
        if (e != cudaSuccess) return e;
        if ((e = launch_pdl(routing_collect_kernel, dim3(1), dim3(1024), 0, stream, st, ro))) return e;
        if ((e = launch_pdl(routing_rank_kernel, dim3((st.max_slots + 255) / 256, RK_SPLIT), dim3(256), 0, stream, st,
                            ro)))
            return e;
        if ((e = launch_pdl(routing_rows_smem_kernel, dim3(1), dim3(1024), sm, stream, st, ro, np2))) return e;
        if ((e = launch_pdl(routing_write_kernel, dim3(st.W), dim3(1024), 0, stream, st, ro))) return e;
    } else {
        if (cudaError_t e = launch_pdl(routing_rows_kernel, dim3(1), dim3(1024), 0, stream, st, ro)) return e;
    }
    return cudaGetLastError();
}

// ------------------------------------------------------------------ K7 (wide): count / scan / scatter
// Block tables per instance, spread over gridDim.y CTAs per instance.  allocate() lays a
// request's pages out member by member in kv order (page_table.cpp:30-45), so instance s's
// pages of a row are its own allocation segment -- pages_for(split) of each earlier member
// in -- followed by whatever append_token grew at the end of the list on s
// (page_table.cpp:86-121).  Only that appended tail is scanned; the segment is a plain copy.
constexpr int RT_SPLIT = 48;
// Segments longer than RT_LONG pages (a 512K-token request has 32K / CP) are copied by a
// whole CTA; shorter ones and every tail by one warp.
constexpr int RT_LONG = 256;

// Row (sl, s): s's allocation segment [seg0, seg1) and the start of the appended tail.
__device__ __forceinline__ void row_segment(const PlannerState& st, int sl, int s, int64_t& seg0, int64_t& seg1,
                                            int64_t& tail0) {
    const int k = st.k[sl];
    int64_t acc = 0;
    seg0 = seg1 = 0;
    for (int m = 0; m < k; ++m) {
        const int64_t need = pages_for_d(st.split[sl * PL_MAXK + m], st.page);
        if (st.kv[sl * PL_MAXK + m] == s) {
            seg0 = acc;
            seg1 = acc + need;
        }
        acc += need;
    }
    tail0 = acc;
}

static __global__ void __launch_bounds__(256) routing_count_kernel(PlannerState st, RoutingOut ro) {
    pdl_trigger();  // K7 launches are PDL-chained (launch_routing_rows / dcp_planner_build_routing)
    pdl_wait();
    const int s = blockIdx.x;
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.y * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int nw = gridDim.y * (blockDim.x >> 5);
    const int S = st.max_slots, W = st.W;
    const int rows = ro.n_count[s];
    int32_t* cu = ro.cu_pages + (size_t)s * (S + 1);
    for (int row = gw; row < rows; row += nw) {  // one warp per row: segment length + tail count
        const int sl = ro.n_slot[(size_t)s * S + row];
        if (lane == 0) ro.n_mrow[(size_t)s * S + row] = ro.slot_mrow[sl];
        int64_t seg0, seg1, tail0;
        row_segment(st, sl, s, seg0, seg1, tail0);
        const int np = st.page_cnt[sl];
        const int64_t off = st.page_off[sl];
        int c = 0;
        for (int64_t t = tail0 + lane; t - lane < np; t += 32)
            c += __popc(__ballot_sync(0xffffffffu, t < np && st.pg_inst[off + t] == s));
        if (lane == 0) cu[row + 1] = static_cast<int>(seg1 - seg0) + c;
    }
    const int mrows = ro.m_count[s];
    const int gt = blockIdx.y * blockDim.x + threadIdx.x;
    for (int row = gt; row < mrows; row += gridDim.y * blockDim.x) {
        const int sl = ro.m_slot[(size_t)s * S + row];
        const int k = st.k[sl];
        ro.m_k[(size_t)s * S + row] = k;
        int32_t* dst = ro.m_nrow + ((size_t)s * S + row) * W;
        for (int c = 0; c < W; ++c) dst[c] = -1;
        for (int m = 0; m < k; ++m) {
            const int sp = st.kv[sl * PL_MAXK + m];
            ro.m_kv[((size_t)s * S + row) * PL_MAXK + m] = sp;
            dst[sp] = ro.slot_nrow[(size_t)sl * W + sp];
        }
    }
}

static __global__ void __launch_bounds__(1024) routing_scan_kernel(PlannerState st, RoutingOut ro) {
    pdl_trigger();  // K7 launches are PDL-chained (launch_routing_rows / dcp_planner_build_routing)
    pdl_wait();
    __shared__ int64_t part[1024];
    const int s = blockIdx.x, tid = threadIdx.x;
    const int S = st.max_slots;
    const int rows = ro.n_count[s];
    int32_t* cu = ro.cu_pages + (size_t)s * (S + 1);
    const int per = (rows + blockDim.x - 1) / blockDim.x;
    int64_t sum = 0;
    for (int j = tid * per; j < min(rows, (tid + 1) * per); ++j) sum += cu[j + 1];
    part[tid] = sum;
    __syncthreads();
    for (int o = 1; o < (int)blockDim.x; o <<= 1) {  // Hillis-Steele inclusive scan
        const int64_t v = tid >= o ? part[tid - o] : 0;
        __syncthreads();
        part[tid] += v;
        __syncthreads();
    }
    int64_t run = part[tid] - sum;
    if (tid == 0) cu[0] = 0;
    for (int j = tid * per; j < min(rows, (tid + 1) * per); ++j) {
        run += cu[j + 1];
        cu[j + 1] = (int32_t)run;
    }
    // the instance's total pages also at the fixed index S (== cu[rows] when rows == S), so K1 can
    // load it together with N instead of after it
    if (tid == blockDim.x - 1 && rows < S) cu[S] = (int32_t)part[tid];
}

static __global__ void __launch_bounds__(256) routing_scatter_kernel(PlannerState st, RoutingOut ro) {
    pdl_trigger();  // K7 launches are PDL-chained (launch_routing_rows / dcp_planner_build_routing)
    pdl_wait();
    const int s = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gw = blockIdx.y * (blockDim.x >> 5) + warp;
    const int nw = gridDim.y * (blockDim.x >> 5);
    const int S = st.max_slots;
    const int rows = ro.n_count[s];
    const int32_t* cu = ro.cu_pages + (size_t)s * (S + 1);
    int32_t* bt = ro.block_table + (size_t)s * st.capacity;
    uint8_t* pf = ro.page_fill + (size_t)s * st.capacity;
    for (int row = gw; row < rows; row += nw) {  // one warp per row: short segment + the tail
        const int sl = ro.n_slot[(size_t)s * S + row];
        int64_t seg0, seg1, tail0;
        row_segment(st, sl, s, seg0, seg1, tail0);
        const int np = st.page_cnt[sl];
        const int64_t off = st.page_off[sl];
        const int segn = static_cast<int>(seg1 - seg0);
        int pos = cu[row];
        if (segn <= RT_LONG) {
            for (int j0 = 0; j0 < segn; j0 += 4 * 32) {
                int fr[4], fi[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int j = j0 + 32 * u + lane;
                    fr[u] = j < segn ? st.pg_frame[off + seg0 + j] : 0;
                    fi[u] = j < segn ? st.pg_fill[off + seg0 + j] : 0;
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int j = j0 + 32 * u + lane;
                    if (j < segn) {
                        bt[pos + j] = fr[u];
                        pf[pos + j] = static_cast<uint8_t>(fi[u]);
                    }
                }
            }
        }
        pos += segn;
        for (int64_t t = tail0 + lane; t - lane < np; t += 32) {
            const bool on = t < np && st.pg_inst[off + t] == s;
            const unsigned b = __ballot_sync(0xffffffffu, on);
            if (on) {
                const int p = pos + __popc(b & ((1u << lane) - 1u));
                bt[p] = st.pg_frame[off + t];
                pf[p] = st.pg_fill[off + t];
            }
            pos += __popc(b);
        }
    }
    for (int row = blockIdx.y; row < rows; row += gridDim.y) {  // long segments: one CTA each, plain copy
        const int sl = ro.n_slot[(size_t)s * S + row];
        int64_t seg0, seg1, tail0;
        row_segment(st, sl, s, seg0, seg1, tail0);
        const int segn = static_cast<int>(seg1 - seg0);
        if (segn <= RT_LONG) continue;
        const int64_t src = st.page_off[sl] + seg0;
        const int pos = cu[row];
        for (int j0 = threadIdx.x; j0 < segn; j0 += 4 * blockDim.x) {
            int fr[4], fi[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int j = j0 + u * blockDim.x;
                fr[u] = j < segn ? st.pg_frame[src + j] : 0;
                fi[u] = j < segn ? st.pg_fill[src + j] : 0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int j = j0 + u * blockDim.x;
                if (j < segn) {
                    bt[pos + j] = fr[u];
                    pf[pos + j] = static_cast<uint8_t>(fi[u]);
                }
            }
        }
    }
}

}  // namespace dcp
