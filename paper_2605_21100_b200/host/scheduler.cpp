// SPDX-License-Identifier: Apache-2.0
//
// dcpsim drop-in: Scheduler::step / rebalance_active / water_fill on the
// device (K6).  The host side synchronises the policy and the FIFO queue into
// the device planner, launches the step kernel, and applies the StepResult,
// the new placements, the rebalanced MoE bindings and the page lists to the
// caller's Request / ClusterState objects (scheduler.cpp:245-306 semantics).
#include <algorithm>
#include <limits>
#include <unordered_map>

#include "dcpsim/scheduler.hpp"

namespace dcpsim {

// ---- configuration helpers (pure arithmetic on the policy) -------------------
int BucketFn::lookup(Tokens seq_len) const {  // scheduler.cpp:10-14
    for (const auto& e : entries)
        if (seq_len <= e.max_len) return e.degree;
    return entries.back().degree;
}

void BucketFn::validate() const {  // scheduler.cpp:16-26
    if (entries.empty()) throw ConfigError("empty bucket table");
    Tokens last_len = 0;
    int last_deg = 0;
    for (const auto& e : entries) {
        if (e.max_len <= last_len) throw ConfigError("bucket lengths must strictly increase");
        if (e.degree < 1 || e.degree < last_deg) throw ConfigError("bucket degrees must be >=1 and non-decreasing");
        last_len = e.max_len;
        last_deg = e.degree;
    }
}

BucketFn BucketFn::default_table() {  // scheduler.cpp:28-33
    BucketFn fn;
    fn.entries = {{32768, 1}, {131072, 2}, {393216, 4}, {std::numeric_limits<Tokens>::max(), 8}};
    return fn;
}

void SchedulerPolicy::validate(const ClusterTopology& topo) const {  // scheduler.cpp:35-41
    if (kind == PolicyKind::DualBalancedDCP) bucket.validate();
    if (kind == PolicyKind::UniformCP && (uniform_degree < 1 || topo.instances_per_node % uniform_degree != 0))
        throw ConfigError("UniformCP degree must divide instances_per_node");
}

int cp_degree(Tokens seq_len, const BucketFn& bucket, int node_instance_count) {
    return std::min(bucket.lookup(seq_len), node_instance_count);
}

bool can_allocate(std::span<const InstanceId> participants, std::span<const Tokens> split,
                  const ClusterState& cluster) {
    for (std::size_t i = 0; i < participants.size(); ++i)
        if (static_cast<std::int64_t>(cluster.instances[static_cast<std::size_t>(participants[i])].free_frames.size()) <
            pages_for(split[i], cluster.topo.page_size))
            return false;
    return true;
}

// ---- device-backed operations ------------------------------------------------
std::vector<Tokens> water_fill(std::span<const InstanceId> participants, Tokens seq_len,
                               std::span<const Tokens> kv_loads) {
    std::vector<Tokens> split(participants.size(), 0);
    if (participants.empty()) return split;
    std::vector<std::int64_t> loads(kv_loads.begin(), kv_loads.begin() + static_cast<long>(participants.size()));
    device::check(dcp_water_fill(device::context(), static_cast<int>(participants.size()), loads.data(), seq_len,
                                 split.data()));
    return split;
}

namespace {

device::Planner& bound_planner(ClusterState& cluster) {
    auto dev = cluster.page_table.device_planner();
    if (!dev) throw ConfigError("ClusterState has no device planner: build it with make_cluster");
    return *dev;
}

void pull_instance_counters(device::Planner& dev, ClusterState& cluster) {
    const int W = dev.world;
    std::vector<std::int64_t> kv(W), nf(W);
    std::vector<std::int32_t> b(W), sc(W);
    device::check(std::min(0, dcp_planner_instances(dev.handle, kv.data(), b.data(), sc.data(), nf.data())));
    for (int s = 0; s < W; ++s) {
        auto& in = cluster.instances[static_cast<std::size_t>(s)];
        in.kv_load = kv[s];
        in.moe_batch = b[s];
        in.shard_count = sc[s];
        if (static_cast<std::int64_t>(in.free_frames.size()) != nf[s])
            throw SimError("host/device free-frame state diverged");
    }
}

void push_policy(device::Planner& dev, const SchedulerPolicy& pol) {
    std::vector<std::int64_t> bl;
    std::vector<std::int32_t> bd;
    for (const auto& e : pol.bucket.entries) {
        bl.push_back(e.max_len);
        bd.push_back(e.degree);
    }
    if (bl.size() > 16) throw ConfigError("bucket tables are limited to 16 entries on the device");
    device::check(dcp_planner_set_policy(dev.handle, static_cast<int>(pol.kind), static_cast<int>(bl.size()),
                                         bl.data(), bd.data(), pol.uniform_degree, pol.hol_strict ? 1 : 0));
}

Placement fetch_placement(device::Planner& dev, RequestId id) {
    std::int32_t kv[64], moe = -1, k = 0;
    std::int64_t split[64];
    device::check(dcp_planner_placement(dev.handle, id, kv, split, &moe, &k));
    Placement p;
    p.moe_binding = moe;
    p.kv_binding.assign(kv, kv + k);
    p.split.assign(split, split + k);
    return p;
}

}  // namespace

void rebalance_active(std::vector<Request*>& active, ClusterState& cluster) {
    auto& dev = bound_planner(cluster);
    std::vector<std::int64_t> ids;
    for (const Request* r : active) ids.push_back(r->id);
    device::check(dcp_planner_rebalance(dev.handle, ids.data(), static_cast<int>(ids.size())));
    // the reference leaves `active` sorted by (cp_degree, id) (scheduler.cpp:45-49)
    std::sort(active.begin(), active.end(), [](const Request* a, const Request* b) {
        const int ka = a->placement->cp_degree(), kb = b->placement->cp_degree();
        return ka != kb ? ka < kb : a->id < b->id;
    });
    const int cap = static_cast<int>(active.size()) + 1024;
    std::vector<std::int64_t> aid(cap);
    std::vector<std::int32_t> amoe(cap);
    const int n = dcp_planner_active_moe(dev.handle, aid.data(), amoe.data(), cap);
    if (n < 0) device::check(n);
    std::unordered_map<std::int64_t, int> moe_of;
    for (int i = 0; i < std::min(n, cap); ++i) moe_of[aid[i]] = amoe[i];
    for (Request* r : active) r->placement->moe_binding = moe_of.at(r->id);
    pull_instance_counters(dev, cluster);
}

StepResult Scheduler::step(std::deque<std::size_t>& waiting, std::span<Request> requests,
                           std::span<const std::size_t> active, ClusterState& cluster) {
    auto& dev = bound_planner(cluster);
    push_policy(dev, policy_);
    // The device recomputes B over its own active set (every committed, unfinished request);
    // the reference recomputes it over `active` (scheduler.cpp:250-261).  They must agree.
    {
        const int acap = static_cast<int>(active.size()) + 1;
        std::vector<std::int64_t> aid(acap);
        std::vector<std::int32_t> amoe(acap);
        const int n = dcp_planner_active_moe(dev.handle, aid.data(), amoe.data(), acap);
        if (n < 0) device::check(n);
        bool same = n == static_cast<int>(active.size());
        if (same) {
            std::vector<std::int64_t> want;
            for (std::size_t idx : active) want.push_back(requests[idx].id);
            std::sort(want.begin(), want.end());
            std::sort(aid.begin(), aid.begin() + n);
            same = std::equal(want.begin(), want.end(), aid.begin());
        }
        if (!same)
            throw InconsistentPlacement("Scheduler::step: `active` differs from the requests committed and not "
                                        "released on this cluster (the device recomputes B over that set)");
    }
    // UniformCP round-robin state belongs to this Scheduler (scheduler.hpp:88), not to the cluster:
    // push it before the round, read it back after (place_uniform, scheduler.cpp:189-222).
    const bool uniform = policy_.kind == PolicyKind::UniformCP;
    if (uniform) {
        const int groups = (cluster.topo.instances_per_node / policy_.uniform_degree) * cluster.topo.nodes;
        if (static_cast<int>(ucp_round_robin_.size()) != groups) ucp_round_robin_.assign(groups, 0);
        device::check(dcp_planner_ucp_rr(dev.handle, ucp_round_robin_.data(), groups, 0));
    }
    // 1. the device queue mirrors the caller's FIFO queue
    std::vector<std::int64_t> ids, lens;
    std::unordered_map<std::int64_t, std::size_t> index_of;
    for (std::size_t idx : waiting) {
        ids.push_back(requests[idx].id);
        lens.push_back(requests[idx].seq_len);
        index_of[requests[idx].id] = idx;
    }
    for (std::size_t idx : active) index_of[requests[idx].id] = idx;
    device::check(dcp_planner_set_queue(dev.handle, ids.data(), lens.data(), static_cast<int>(ids.size())));
    // 2. one scheduling round on the device (K6)
    device::check(dcp_planner_step(dev.handle, nullptr));
    const std::size_t cap = ids.size() + 1;
    std::vector<std::int64_t> c(cap), d(cap), u(cap);
    std::int32_t nc = 0, nd = 0, nu = 0;
    std::int64_t hol = 0;
    device::check(dcp_planner_step_result(dev.handle, c.data(), &nc, d.data(), &nd, u.data(), &nu, &hol));
    StepResult res;
    res.committed.assign(c.begin(), c.begin() + nc);
    res.deferred.assign(d.begin(), d.begin() + nd);
    res.unschedulable.assign(u.begin(), u.begin() + nu);
    res.hol_events = hol;
    if (uniform)
        device::check(dcp_planner_ucp_rr(dev.handle, ucp_round_robin_.data(),
                                         static_cast<int>(ucp_round_robin_.size()), 1));
    // 3. rebalanced MoE bindings of the active set (DCP) / sticky otherwise
    if (policy_.kind == PolicyKind::DualBalancedDCP && !active.empty()) {
        const int acap = static_cast<int>(active.size() + res.committed.size()) + 1024;
        std::vector<std::int64_t> aid(acap);
        std::vector<std::int32_t> amoe(acap);
        const int n = dcp_planner_active_moe(dev.handle, aid.data(), amoe.data(), acap);
        if (n < 0) device::check(n);
        for (int i = 0; i < std::min(n, acap); ++i) {
            auto it = index_of.find(aid[i]);
            if (it != index_of.end() && requests[it->second].placement)
                requests[it->second].placement->moe_binding = amoe[i];
        }
    }
    // 4. committed requests: placement, page list, LIFO pops on the host mirror
    for (RequestId id : res.committed) {
        Request& r = requests[index_of.at(id)];
        r.placement = fetch_placement(dev, id);
        r.state = RequestState::Active;
        cluster.page_table.mirror_allocation(id, *r.placement, cluster.instances);
    }
    pull_instance_counters(dev, cluster);
    // 5. the caller's queue loses committed and unschedulable entries, in order
    std::unordered_map<std::int64_t, int> gone;
    for (auto id : res.committed) gone[id] = 1;
    for (auto id : res.unschedulable) gone[id] = 1;
    std::deque<std::size_t> kept;
    for (std::size_t idx : waiting)
        if (!gone.count(requests[idx].id)) kept.push_back(idx);
    waiting.swap(kept);
    return res;
}

}  // namespace dcpsim
