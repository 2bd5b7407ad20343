// SPDX-License-Identifier: Apache-2.0
//
// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// POD C wrapper around the *unmodified* reference library
// (/root/reference/proj, compiled from where it lies by oracle/Makefile with
// -Ddcpsim=dcpsim_ref) so tests, smoke() and bench.py's reference arm can call
// the reference's own code through ctypes.  Output: oracle/_ref/libdcpsim_ref.so
// (git-ignored, shipped to the GPU box by gpurun).  Nothing here re-implements
// reference behaviour; every function forwards to the dcpsim_ref:: symbol named
// in its comment.
#include <chrono>
#include <omp.h>

#include <cstdint>
#include <cstring>
#include <deque>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "dcpsim/attn_merge.hpp"
#include "dcpsim/page_table.hpp"
#include "dcpsim/routing.hpp"
#include "dcpsim/scheduler.hpp"
#include "dcpsim/types.hpp"
#include "dcpsim/workload.hpp"

namespace R = dcpsim;  // renamed to dcpsim_ref by -Ddcpsim=dcpsim_ref

namespace {

// Map reference exceptions onto the C-ABI codes of include/dcp_capi.h.
template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const R::InsufficientFrames&) {
        return -1;
    } catch (const R::UnknownRequest&) {
        return -2;
    } catch (const R::UnknownPage&) {
        return -3;
    } catch (const R::InconsistentPlacement&) {
        return -4;
    } catch (const R::ShapeOverflow&) {
        return -5;
    } catch (const R::EmptyShard&) {
        return -6;
    } catch (const R::ConfigError&) {
        return -7;
    } catch (...) {
        return -100;
    }
}

int copy_string(const std::string& s, char* buf, int64_t cap) {
    if (buf && cap > 0) {
        const auto n = static_cast<int64_t>(s.size()) < cap - 1 ? s.size() : static_cast<size_t>(cap - 1);
        std::memcpy(buf, s.data(), n);
        buf[n] = 0;
    }
    return static_cast<int>(s.size());
}

struct World {
    R::ClusterState cluster;
    std::unique_ptr<R::Scheduler> sched;
    std::vector<R::Request> requests;   // index = insertion order
    std::deque<std::size_t> waiting;
    R::StepResult last;
};

R::SchedulerPolicy make_policy(int kind, const int64_t* bucket_len, const int* bucket_deg,
                               int n_bucket, int uniform_degree, int hol_strict) {
    R::SchedulerPolicy pol;
    pol.kind = static_cast<R::PolicyKind>(kind);
    if (n_bucket > 0) {
        pol.bucket.entries.clear();
        for (int i = 0; i < n_bucket; ++i) pol.bucket.entries.push_back({bucket_len[i], bucket_deg[i]});
    }
    pol.uniform_degree = uniform_degree;
    pol.hol_strict = hol_strict != 0;
    return pol;
}

}  // namespace

extern "C" {

// ---------------------------------------------------------------- attention
// dcpsim::shard_attention<T> (attn_merge.hpp:53-82)
int dcpref_shard_attention_f64(const double* q, const double* k, const double* v, int64_t len,
                               int d, double scale, double* out, double* lse) {
    return guarded([&] {
        auto r = R::shard_attention<double>({q, (size_t)d}, {k, (size_t)(len * d)},
                                            {v, (size_t)(len * d)}, len, d, scale);
        std::memcpy(out, r.partial_out.data(), sizeof(double) * d);
        *lse = r.lse;
    });
}
int dcpref_shard_attention_f32(const float* q, const float* k, const float* v, int64_t len, int d,
                               float scale, float* out, float* lse) {
    return guarded([&] {
        auto r = R::shard_attention<float>({q, (size_t)d}, {k, (size_t)(len * d)},
                                           {v, (size_t)(len * d)}, len, d, scale);
        std::memcpy(out, r.partial_out.data(), sizeof(float) * d);
        *lse = r.lse;
    });
}
// dcpsim::reference_attention<T> (attn_merge.hpp:25-50)
int dcpref_reference_attention_f64(const double* q, const double* k, const double* v, int64_t len,
                                   int d, double scale, double* out) {
    return guarded([&] {
        auto r = R::reference_attention<double>({q, (size_t)d}, {k, (size_t)(len * d)},
                                                {v, (size_t)(len * d)}, len, d, scale);
        std::memcpy(out, r.data(), sizeof(double) * d);
    });
}
// dcpsim::lse_merge<T> (attn_merge.hpp:86-100); partials in list order.
int dcpref_lse_merge_f64(int n, const double* outs, const double* lses, int d, double* out) {
    return guarded([&] {
        std::vector<R::AttnShardResult<double>> ps(n);
        for (int i = 0; i < n; ++i) {
            ps[i].partial_out.assign(outs + (size_t)i * d, outs + (size_t)(i + 1) * d);
            ps[i].lse = lses[i];
        }
        auto r = R::lse_merge<double>(ps);
        std::memcpy(out, r.data(), sizeof(double) * d);
    });
}
// dcpsim::sharded_attention_merge (attn_merge.cpp:64-77)
int dcpref_sharded_attention_merge_f32(const float* q, const float* k, const float* v, int64_t len,
                                       int d, float scale, const int64_t* bounds, int nb,
                                       int parallel, float* out) {
    return guarded([&] {
        auto r = R::sharded_attention_merge({q, (size_t)d}, {k, (size_t)(len * d)},
                                            {v, (size_t)(len * d)}, d, scale,
                                            {bounds, (size_t)nb}, parallel != 0);
        std::memcpy(out, r.data(), sizeof(float) * d);
    });
}
int dcpref_sharded_attention_merge_f64(const double* q, const double* k, const double* v,
                                       int64_t len, int d, double scale, const int64_t* bounds,
                                       int nb, int parallel, double* out) {
    return guarded([&] {
        auto r = R::sharded_attention_merge({q, (size_t)d}, {k, (size_t)(len * d)},
                                            {v, (size_t)(len * d)}, d, scale,
                                            {bounds, (size_t)nb}, parallel != 0);
        std::memcpy(out, r.data(), sizeof(double) * d);
    });
}

// CPU baseline driver for the decode-attention step: an
// outer OpenMP loop over (request, q-head) calling the reference's
// sharded_attention_merge(parallel=false) on contiguous fp32 K/V that the
// caller gathered per (request, kv-head) in logical page order.
//   q      [nreq][hq][d]         k,v: per request r, kv head j at
//   kv_off[r] + j*len[r]*d       (fp32, contiguous [len][d])
//   bounds per request: nbounds[r] entries starting at bounds_off[r]
int dcpref_batch_decode_attn_f32(int nreq, int hq, int hkv, int d, float scale, const float* q,
                                 const float* k, const float* v, const int64_t* kv_off,
                                 const int64_t* len, const int64_t* bounds,
                                 const int64_t* bounds_off, const int* nbounds, float* out,
                                 int threads) {
    const int group = hq / hkv;
    int rc = 0;
    if (threads > 0) omp_set_num_threads(threads);
#pragma omp parallel for schedule(dynamic) reduction(min : rc)
    for (int64_t w = 0; w < (int64_t)nreq * hq; ++w) {
        const int r = (int)(w / hq), h = (int)(w % hq), j = h / group;
        const size_t base = (size_t)kv_off[r] + (size_t)j * len[r] * d;
        int e = guarded([&] {
            auto o = R::sharded_attention_merge(
                {q + ((size_t)r * hq + h) * d, (size_t)d}, {k + base, (size_t)(len[r] * d)},
                {v + base, (size_t)(len[r] * d)}, d, scale,
                {bounds + bounds_off[r], (size_t)nbounds[r]}, false);
            std::memcpy(out + ((size_t)r * hq + h) * d, o.data(), sizeof(float) * d);
        });
        rc = e < rc ? e : rc;
    }
    return rc;
}

// ---------------------------------------------------------------- planner pieces
// dcpsim::water_fill (scheduler.cpp:70-102)
int dcpref_water_fill(int n, const int32_t* participants, int64_t seq_len, const int64_t* loads,
                      int64_t* split) {
    return guarded([&] {
        auto s = R::water_fill({participants, (size_t)n}, seq_len, {loads, (size_t)n});
        std::memcpy(split, s.data(), sizeof(int64_t) * n);
    });
}
// dcpsim::cp_degree + BucketFn::lookup (scheduler.cpp:10-14, 66-68); n_bucket==0 → default_table
int dcpref_cp_degree(int64_t seq_len, const int64_t* bucket_len, const int* bucket_deg,
                     int n_bucket, int node_instances) {
    R::BucketFn fn = R::BucketFn::default_table();
    if (n_bucket > 0) {
        fn.entries.clear();
        for (int i = 0; i < n_bucket; ++i) fn.entries.push_back({bucket_len[i], bucket_deg[i]});
    }
    return R::cp_degree(seq_len, fn, node_instances);
}
// dcpsim::bucket_shape on ShapeSpace::default_space() (routing.cpp:89-109)
int dcpref_bucket_shape_default(int m, int n, int* bm, int* bn) {
    return guarded([&] {
        auto r = R::bucket_shape(m, n, R::ShapeSpace::default_space());
        *bm = r.first;
        *bn = r.second;
    });
}
// dcpsim::graph_memory_footprint (routing.cpp:111-127) on the default space with overrides
int dcpref_graph_footprint(int world, int heads, int head_size, int hidden, int max_blocks,
                           int elem, int idx, int64_t* graphs, int64_t* bytes) {
    return guarded([&] {
        auto s = R::ShapeSpace::default_space();
        s.world_size = world;
        s.num_heads = heads;
        s.head_size = head_size;
        s.hidden_dim = hidden;
        s.max_blocks = max_blocks;
        s.element_size = elem;
        s.index_size = idx;
        auto f = R::graph_memory_footprint(s);
        *graphs = f.graph_count;
        *bytes = f.buffer_bytes;
    });
}

// ---------------------------------------------------------------- world (scheduler + cluster)
void* dcpref_world_create(int nodes, int inst_per_node, int64_t page_size, int64_t capacity,
                          int kind, const int64_t* bucket_len, const int* bucket_deg, int n_bucket,
                          int uniform_degree, int hol_strict) {
    auto* w = new World();
    R::ClusterTopology topo;
    topo.nodes = nodes;
    topo.instances_per_node = inst_per_node;
    topo.page_size = page_size;
    w->cluster = R::make_cluster(topo, capacity);
    auto pol = make_policy(kind, bucket_len, bucket_deg, n_bucket, uniform_degree, hol_strict);
    w->sched = std::make_unique<R::Scheduler>(pol);
    return w;
}
void dcpref_world_destroy(void* h) { delete static_cast<World*>(h); }

// Append a request at the back of the FIFO waiting queue.
int dcpref_world_enqueue(void* h, int64_t id, int64_t seq_len) {
    auto* w = static_cast<World*>(h);
    R::Request r;
    r.id = id;
    r.seq_len = seq_len;
    w->requests.push_back(r);
    w->waiting.push_back(w->requests.size() - 1);
    return 0;
}

// dcpsim::Scheduler::step (scheduler.cpp:245-306) with the active set = all
// Active requests in insertion order.  Output arrays sized by caller (>= #requests).
int dcpref_world_step(void* h, int64_t* committed, int* n_committed, int64_t* deferred,
                      int* n_deferred, int64_t* unsched, int* n_unsched, int64_t* hol) {
    auto* w = static_cast<World*>(h);
    std::vector<std::size_t> active;
    for (std::size_t i = 0; i < w->requests.size(); ++i)
        if (w->requests[i].state == R::RequestState::Active) active.push_back(i);
    return guarded([&] {
        w->last = w->sched->step(w->waiting, w->requests, active, w->cluster);
        *n_committed = (int)w->last.committed.size();
        *n_deferred = (int)w->last.deferred.size();
        *n_unsched = (int)w->last.unschedulable.size();
        for (size_t i = 0; i < w->last.committed.size(); ++i) committed[i] = w->last.committed[i];
        for (size_t i = 0; i < w->last.deferred.size(); ++i) deferred[i] = w->last.deferred[i];
        for (size_t i = 0; i < w->last.unschedulable.size(); ++i) unsched[i] = w->last.unschedulable[i];
        *hol = w->last.hol_events;
    });
}

static R::Request* find_req(World* w, int64_t id) {
    for (auto& r : w->requests)
        if (r.id == id) return &r;
    return nullptr;
}

// dcpsim::pt_free (page_table.cpp:51-66, 156-158) + mark Finished.
int dcpref_world_finish(void* h, int64_t id) {
    auto* w = static_cast<World*>(h);
    return guarded([&] {
        R::pt_free(id, w->cluster);
        if (auto* r = find_req(w, id)) {
            r->state = R::RequestState::Finished;
        }
    });
}

// dcpsim::GlobalPageTable::append_token (page_table.cpp:86-121)
int dcpref_world_append_token(void* h, int64_t id, int32_t* instance) {
    auto* w = static_cast<World*>(h);
    return guarded([&] {
        auto* r = find_req(w, id);
        if (!r || !r->placement) throw R::UnknownRequest("no placement");
        *instance = w->cluster.page_table.append_token(id, *r->placement, w->cluster.instances);
        if (*instance >= 0) r->generated += 1;
    });
}

int dcpref_world_placement(void* h, int64_t id, int32_t* kv, int64_t* split, int32_t* moe,
                           int* k) {
    auto* w = static_cast<World*>(h);
    auto* r = find_req(w, id);
    if (!r || !r->placement) return -2;
    const auto& p = *r->placement;
    *k = p.cp_degree();
    *moe = p.moe_binding;
    for (int i = 0; i < *k; ++i) {
        kv[i] = p.kv_binding[i];
        split[i] = p.split[i];
    }
    return 0;
}

int dcpref_world_instances(void* h, int64_t* kv_load, int32_t* moe_batch, int32_t* shard_count,
                           int64_t* free_frames) {
    auto* w = static_cast<World*>(h);
    for (size_t i = 0; i < w->cluster.instances.size(); ++i) {
        const auto& s = w->cluster.instances[i];
        kv_load[i] = s.kv_load;
        moe_batch[i] = s.moe_batch;
        shard_count[i] = s.shard_count;
        free_frames[i] = (int64_t)s.free_frames.size();
    }
    return (int)w->cluster.instances.size();
}

// dcpsim::GlobalPageTable::dump_csv (page_table.cpp:123-131)
int dcpref_world_dump_page_table(void* h, char* buf, int64_t cap) {
    auto* w = static_cast<World*>(h);
    std::ostringstream os;
    w->cluster.page_table.dump_csv(os);
    return copy_string(os.str(), buf, cap);
}

// build_binding_config + derive_routing_tables + dump_routing_csv (routing.cpp:9-79)
// over the Active requests.
int dcpref_world_dump_routing(void* h, char* buf, int64_t cap) {
    auto* w = static_cast<World*>(h);
    std::vector<const R::Request*> act;
    for (auto& r : w->requests)
        if (r.state == R::RequestState::Active) act.push_back(&r);
    std::string s;
    int rc = guarded([&] {
        auto cfg = R::build_binding_config(act, w->cluster.topo.world_size());
        auto rt = R::derive_routing_tables(cfg);
        std::ostringstream os;
        R::dump_routing_csv(rt, os);
        s = os.str();
    });
    if (rc) return rc;
    return copy_string(s, buf, cap);
}

// Timing of the reference's routing build alone: build_binding_config + derive_routing_tables
// (routing.cpp:9-63) over the Active requests, no CSV; best of `reps` in nanoseconds.
int dcpref_world_time_routing(void* h, int reps, int64_t* best_ns) {
    auto* w = static_cast<World*>(h);
    std::vector<const R::Request*> act;
    for (auto& r : w->requests)
        if (r.state == R::RequestState::Active) act.push_back(&r);
    int64_t best = INT64_MAX;
    size_t sink = 0;
    int rc = guarded([&] {
        for (int i = 0; i < reps; ++i) {
            const auto t0 = std::chrono::steady_clock::now();
            auto cfg = R::build_binding_config(act, w->cluster.topo.world_size());
            auto rt = R::derive_routing_tables(cfg);
            const auto t1 = std::chrono::steady_clock::now();
            sink += rt.size();
            best = std::min<int64_t>(best, std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count());
        }
    });
    *best_ns = sink ? best : best;
    return rc;
}

// dcpsim::uniform_int / mt19937_64 (workload.hpp:18-26): n draws in [lo, hi].
void dcpref_uniform_int(uint64_t seed, int64_t lo, int64_t hi, int n, int64_t* out) {
    std::mt19937_64 rng(seed);
    for (int i = 0; i < n; ++i) out[i] = R::uniform_int(rng, lo, hi);
}

// dcpsim::gen_trace (workload.cpp:73-106) with the shipped distributions.
int dcpref_gen_trace(uint64_t seed, double long_ratio, double rate, double duration_s,
                     int poisson, int64_t* ids, int64_t* seq_len, double* arrival_ms,
                     int64_t* out_len, int cap) {
    R::TraceConfig c;
    c.short_dist = R::sharegpt4o_distribution();
    c.long_dist = R::github_issue_distribution();
    c.long_ratio = long_ratio;
    c.arrival.kind = poisson ? R::ArrivalKind::Poisson : R::ArrivalKind::ConstantRate;
    c.arrival.rate_per_s = rate;
    c.duration_s = duration_s;
    c.seed = seed;
    std::vector<R::Request> t;
    int rc = guarded([&] { t = R::gen_trace(c); });
    if (rc) return rc;
    const int n = (int)t.size() < cap ? (int)t.size() : cap;
    for (int i = 0; i < n; ++i) {
        ids[i] = t[i].id;
        seq_len[i] = t[i].seq_len;
        arrival_ms[i] = t[i].arrival_ms;
        out_len[i] = t[i].output_len;
    }
    return (int)t.size();
}

// dcpsim::gen_trace + dcpsim::write_trace_csv (workload.cpp:108-115): the CSV text of a
// generated trace; returns the full length (copies at most cap-1 bytes + NUL).
int64_t dcpref_trace_csv(uint64_t seed, double long_ratio, double rate, double duration_s, int poisson,
                         char* buf, int64_t cap) {
    R::TraceConfig c;
    c.short_dist = R::sharegpt4o_distribution();
    c.long_dist = R::github_issue_distribution();
    c.long_ratio = long_ratio;
    c.arrival.kind = poisson ? R::ArrivalKind::Poisson : R::ArrivalKind::ConstantRate;
    c.arrival.rate_per_s = rate;
    c.duration_s = duration_s;
    c.seed = seed;
    std::ostringstream os;
    int rc = guarded([&] { R::write_trace_csv(R::gen_trace(c), os); });
    if (rc) return rc;
    return copy_string(os.str(), buf, cap);
}

// dcpsim::load_trace_csv (workload.cpp:117-137) over CSV text; returns the request count
// (fills at most cap) or a negative error code (ConfigError for an empty file).
int dcpref_load_trace_csv(const char* text, int64_t* ids, double* arrival_ms, int64_t* seq_len,
                          int64_t* out_len, int cap) {
    std::vector<R::Request> t;
    int rc = guarded([&] {
        std::istringstream is(text);
        t = R::load_trace_csv(is);
    });
    if (rc) return rc;
    const int n = (int)t.size() < cap ? (int)t.size() : cap;
    for (int i = 0; i < n; ++i) {
        ids[i] = t[i].id;
        arrival_ms[i] = t[i].arrival_ms;
        seq_len[i] = t[i].seq_len;
        out_len[i] = t[i].output_len;
    }
    return (int)t.size();
}

}  // extern "C"
