// SPDX-License-Identifier: Apache-2.0
//
// dcpsim drop-in: GlobalPageTable / ClusterState over the device planner.
// Every mutation (allocate, release, append_token) is executed by a K6
// kernel on the cluster's device planner (LIFO frame stacks in HBM); this
// file only applies the device's answer to the host mirror the reference API
// exposes (page_table.cpp:9-158 semantics) and checks the two agree.
#include <algorithm>
#include <cstdlib>
#include <memory>
#include <string>

#include "dcpsim/page_table.hpp"

namespace dcpsim {

namespace {

std::shared_ptr<device::Planner> create_planner(int nodes, int ipn, Tokens page, std::int64_t capacity) {
    dcp_planner_config cfg{};
    cfg.nodes = nodes;
    cfg.instances_per_node = ipn;
    cfg.page_size = page;
    cfg.capacity_pages = capacity;
    cfg.policy = DCP_POLICY_DCP;
    cfg.n_bucket = 0;
    cfg.uniform_degree = 1;
    cfg.hol_strict = 1;
    const char* e = std::getenv("DCPSIM_MAX_REQUESTS");
    cfg.max_requests = e ? std::atoi(e) : 16384;
    cfg.reserve_pages = 4;
    auto p = std::make_shared<device::Planner>();
    device::check(dcp_planner_create(device::context(), &cfg, &p->handle));
    p->world = nodes * ipn;
    p->page_size = page;
    p->capacity = capacity;
    return p;
}

}  // namespace

ClusterState make_cluster(const ClusterTopology& topo, std::int64_t capacity) {
    ClusterState c;
    c.topo = topo;
    c.instances.resize(static_cast<std::size_t>(topo.world_size()));
    for (int s = 0; s < topo.world_size(); ++s) {
        auto& inst = c.instances[static_cast<std::size_t>(s)];
        inst.id = s;
        inst.node = topo.node_of(s);
        inst.capacity_pages = capacity;
        inst.free_frames.resize(static_cast<std::size_t>(capacity));
        for (std::int64_t f = 0; f < capacity; ++f)  // top of the stack = lowest frame id
            inst.free_frames[static_cast<std::size_t>(f)] = capacity - 1 - f;
    }
    c.page_table.bind_device(create_planner(topo.nodes, topo.instances_per_node, topo.page_size, capacity));
    return c;
}

device::Planner& GlobalPageTable::ensure_device(const std::vector<InstanceState>& instances, Tokens page_size) {
    if (dev_) {
        if (dev_->page_size != page_size)
            throw ConfigError("page_size " + std::to_string(page_size) + " differs from the bound cluster's " +
                              std::to_string(dev_->page_size));
        return *dev_;
    }
    // Standalone table: bind a planner loaded with the host instance state.
    if (!entries_.empty()) throw ConfigError("cannot bind a non-empty page table to the device");
    const int W = static_cast<int>(instances.size());
    const std::int64_t cap = instances.empty() ? 0 : instances.front().capacity_pages;
    auto p = create_planner(W, 1, page_size, cap);
    std::vector<std::int64_t> kv(W), nf(W);
    std::vector<std::int32_t> b(W), sc(W), stacks(static_cast<std::size_t>(W) * cap);
    for (int s = 0; s < W; ++s) {
        const auto& in = instances[static_cast<std::size_t>(s)];
        if (in.capacity_pages != cap) throw ConfigError("instances must share one capacity");
        kv[s] = in.kv_load;
        b[s] = in.moe_batch;
        sc[s] = in.shard_count;
        nf[s] = static_cast<std::int64_t>(in.free_frames.size());
        for (std::size_t i = 0; i < in.free_frames.size(); ++i)
            stacks[static_cast<std::size_t>(s) * cap + i] = static_cast<std::int32_t>(in.free_frames[i]);
    }
    device::check(dcp_planner_load_instances(p->handle, kv.data(), b.data(), sc.data(), nf.data(), stacks.data()));
    dev_ = p;
    return *dev_;
}

// Apply a device allocation to the host mirror: the device popped the tops of
// the same LIFO stacks, so the host pops must yield the same frame ids.
void GlobalPageTable::mirror_allocation(RequestId id, const Placement& p, std::vector<InstanceState>& instances) {
    auto& dev = *dev_;
    const std::int64_t n = dcp_planner_pages(dev.handle, id, nullptr, nullptr, 0);
    if (n < 0) device::check(static_cast<int>(n));
    std::vector<std::int32_t> inst(static_cast<std::size_t>(n)), frame(static_cast<std::size_t>(n));
    dcp_planner_pages(dev.handle, id, inst.data(), frame.data(), n);
    Entry e;
    e.page_size = dev.page_size;
    for (std::int64_t i = 0; i < n; ++i) {
        auto& fl = instances[static_cast<std::size_t>(inst[i])].free_frames;
        if (fl.empty() || fl.back() != frame[i])
            throw SimError("host/device page-table state diverged (mutate the cluster only via dcpsim)");
        fl.pop_back();
        e.pages.push_back(PageRef{inst[i], frame[i]});
    }
    for (std::size_t m = 0; m < p.kv_binding.size(); ++m) {
        const InstanceId s = p.kv_binding[m];
        instances[static_cast<std::size_t>(s)].kv_load += p.split[m];
        e.shard_tokens[s] += p.split[m];
        if (p.split[m] > 0) {
            const Tokens r = p.split[m] % dev.page_size;
            e.trailing_fill = r == 0 ? dev.page_size : r;
        }
    }
    entries_[id] = std::move(e);
}

const std::vector<PageRef>& GlobalPageTable::allocate(const Request& request, const Placement& placement,
                                                      Tokens page_size, std::vector<InstanceState>& instances) {
    if (entries_.count(request.id)) throw InsufficientFrames("request already has page-table entries");
    if (request.seq_len < 1) throw InsufficientFrames("cannot allocate a zero-length request");
    if (placement.split.size() != placement.kv_binding.size())
        throw InconsistentPlacement("kv_binding/split size mismatch");
    auto& dev = ensure_device(instances, page_size);
    std::vector<std::int32_t> kv(placement.kv_binding.begin(), placement.kv_binding.end());
    device::check(dcp_planner_allocate(dev.handle, request.id, request.seq_len, static_cast<int>(kv.size()),
                                       kv.data(), placement.split.data(), placement.moe_binding));
    mirror_allocation(request.id, placement, instances);
    return entries_[request.id].pages;
}

std::vector<std::pair<InstanceId, std::int64_t>> GlobalPageTable::release(RequestId id,
                                                                          std::vector<InstanceState>& instances) {
    auto it = entries_.find(id);
    if (it == entries_.end()) throw UnknownRequest("no page-table entries for request " + std::to_string(id));
    device::check(dcp_planner_finish(dev_->handle, &id, 1, nullptr));
    std::map<InstanceId, std::int64_t> released;
    for (const auto& p : it->second.pages) {
        instances[static_cast<std::size_t>(p.instance)].free_frames.push_back(p.frame);
        released[p.instance] += 1;
    }
    for (const auto& [s, t] : it->second.shard_tokens) instances[static_cast<std::size_t>(s)].kv_load -= t;
    entries_.erase(it);
    return {released.begin(), released.end()};
}

PageRef GlobalPageTable::lookup(RequestId id, std::int64_t logical_page) const {
    auto it = entries_.find(id);
    if (it == entries_.end()) throw UnknownPage("unknown request " + std::to_string(id));
    const auto& pages = it->second.pages;
    if (logical_page < 0 || logical_page >= static_cast<std::int64_t>(pages.size()))
        throw UnknownPage("logical page " + std::to_string(logical_page) + " out of range for request " +
                          std::to_string(id));
    return pages[static_cast<std::size_t>(logical_page)];
}

std::int64_t GlobalPageTable::page_count(RequestId id) const {
    auto it = entries_.find(id);
    if (it == entries_.end()) throw UnknownRequest("no page-table entries for request " + std::to_string(id));
    return static_cast<std::int64_t>(it->second.pages.size());
}

InstanceId GlobalPageTable::append_token(RequestId id, const Placement&, std::vector<InstanceState>& instances) {
    auto it = entries_.find(id);
    if (it == entries_.end()) throw UnknownRequest("no page-table entries for request " + std::to_string(id));
    std::int32_t target = -1;
    device::check(dcp_planner_append_token(dev_->handle, &id, 1, &target));
    if (target < 0) return -1;  // growth stall
    Entry& e = it->second;
    auto& inst = instances[static_cast<std::size_t>(target)];
    if (!e.pages.empty() && e.trailing_fill < e.page_size) {
        e.trailing_fill += 1;  // device filled the trailing slot of the last page
    } else {
        if (inst.free_frames.empty()) throw SimError("host/device page-table state diverged");
        e.pages.push_back(PageRef{target, inst.free_frames.back()});
        inst.free_frames.pop_back();
        e.trailing_fill = 1;
    }
    inst.kv_load += 1;
    e.shard_tokens[target] += 1;
    return target;
}

void GlobalPageTable::dump_csv(std::ostream& out) const {
    out << "request_id,logical_page,instance_id,frame_id\n";
    for (const auto& [id, e] : entries_)
        for (std::size_t p = 0; p < e.pages.size(); ++p)
            out << id << ',' << p << ',' << e.pages[p].instance << ',' << e.pages[p].frame << '\n';
}

const std::vector<PageRef>& pt_allocate(const Request& request, const Placement& placement, ClusterState& cluster) {
    return cluster.page_table.allocate(request, placement, cluster.topo.page_size, cluster.instances);
}

std::vector<std::pair<InstanceId, std::int64_t>> pt_free(RequestId id, ClusterState& cluster) {
    return cluster.page_table.release(id, cluster.instances);
}

PageRef pt_lookup(const ClusterState& cluster, RequestId id, std::int64_t logical_page) {
    return cluster.page_table.lookup(id, logical_page);
}

}  // namespace dcpsim
