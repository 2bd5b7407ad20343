// SPDX-License-Identifier: Apache-2.0
//
// dcpsim drop-in: build_binding_config / derive_routing_tables on the device
// (K7 routing_rows_kernel, route expansion kernel), CSV writer, ShapeSpace
// configuration helpers (routing.cpp:9-127 semantics).
#include <algorithm>
#include <string>

#include "dcpsim/device.hpp"
#include "dcpsim/routing.hpp"

namespace dcpsim {

std::vector<BindingConfig> build_binding_config(std::span<const Request* const> active, int world_size) {
    const int n = static_cast<int>(active.size());
    std::vector<std::int64_t> ids(n);
    std::vector<std::int32_t> k(n), moe(n), kv(static_cast<std::size_t>(n) * 16, 0);
    for (int i = 0; i < n; ++i) {
        const Request* r = active[static_cast<std::size_t>(i)];
        const Placement& p = *r->placement;
        if (p.kv_binding.size() > 16) throw ConfigError("cp_degree > 16 is not supported on the device");
        ids[i] = r->id;
        k[i] = p.cp_degree();
        moe[i] = p.moe_binding;
        for (int m = 0; m < k[i]; ++m) kv[static_cast<std::size_t>(i) * 16 + m] = p.kv_binding[m];
    }
    std::vector<std::int32_t> nc(world_size), mc(world_size);
    std::vector<std::int32_t> nrows(static_cast<std::size_t>(world_size) * std::max(n, 1)),
        mrows(static_cast<std::size_t>(world_size) * std::max(n, 1));
    device::check(dcp_binding_config(device::context(), n, ids.data(), k.data(), moe.data(), kv.data(), world_size,
                                     nc.data(), mc.data(), nrows.data(), mrows.data()));
    std::vector<BindingConfig> cfg(static_cast<std::size_t>(world_size));
    for (int s = 0; s < world_size; ++s) {
        auto& c = cfg[static_cast<std::size_t>(s)];
        for (int j = 0; j < mc[s]; ++j) {
            const Request* r = active[static_cast<std::size_t>(mrows[static_cast<std::size_t>(s) * n + j])];
            c.moe_bound.push_back(r->id);
            c.moe_bound_kv.push_back(r->placement->kv_binding);
        }
        for (int j = 0; j < nc[s]; ++j) {
            const Request* r = active[static_cast<std::size_t>(nrows[static_cast<std::size_t>(s) * n + j])];
            c.shard_requests.push_back(r->id);
            c.shard_request_moe.push_back(r->placement->moe_binding);
        }
    }
    return cfg;
}

std::vector<InstanceRouting> derive_routing_tables(std::span<const BindingConfig> configs) {
    const int W = static_cast<int>(configs.size());
    std::vector<InstanceRouting> out(configs.size());
    for (int s = 0; s < W; ++s) {
        const auto& c = configs[static_cast<std::size_t>(s)];
        std::vector<std::uint32_t> mask(static_cast<std::size_t>(c.m()));
        for (int r = 0; r < c.m(); ++r)
            for (InstanceId x : c.moe_bound_kv[static_cast<std::size_t>(r)]) mask[static_cast<std::size_t>(r)] |= 1u << x;
        std::vector<std::int32_t> sm(c.shard_request_moe.begin(), c.shard_request_moe.end());
        auto& q = out[static_cast<std::size_t>(s)].q_route;
        auto& res = out[static_cast<std::size_t>(s)].res_route;
        q.rows = c.n();
        q.cols = W;
        q.bits.assign(static_cast<std::size_t>(c.n()) * W, 0);
        q.row_requests = c.shard_requests;
        res.rows = c.m();
        res.cols = W;
        res.bits.assign(static_cast<std::size_t>(c.m()) * W, 0);
        res.row_requests = c.moe_bound;
        device::check(dcp_route_tables(device::context(), W, c.n(), sm.data(), c.m(), mask.data(), q.bits.data(),
                                       res.bits.data()));
    }
    return out;
}

void dump_routing_csv(std::span<const InstanceRouting> routing, std::ostream& out) {
    out << "instance,table,row,request_id,columns\n";
    for (std::size_t i = 0; i < routing.size(); ++i) {
        for (int t = 0; t < 2; ++t) {
            const RouteTable& tab = t == 0 ? routing[i].q_route : routing[i].res_route;
            for (int r = 0; r < tab.rows; ++r) {
                out << i << ',' << (t == 0 ? "q_route" : "res_route") << ',' << r << ','
                    << tab.row_requests[static_cast<std::size_t>(r)] << ',';
                for (int c = 0; c < tab.cols; ++c) out << static_cast<int>(tab.at(r, c));
                out << '\n';
            }
        }
    }
}

void ShapeSpace::validate() const {
    if (buckets.empty()) return;
    if (!std::is_sorted(buckets.begin(), buckets.end())) throw ConfigError("shape buckets must be sorted");
    if (std::find(buckets.begin(), buckets.end(), std::make_pair(m_max, n_max)) == buckets.end())
        throw ConfigError("shape space must contain (m_max, n_max)");
}

ShapeSpace ShapeSpace::default_space() {  // 6 x 8 = 48 buckets (routing.cpp:89-99)
    ShapeSpace sp;
    for (int m : {8, 16, 32, 64, 128, 256})
        for (int n : {8, 16, 32, 64, 128, 256, 384, 512}) sp.buckets.emplace_back(m, n);
    std::sort(sp.buckets.begin(), sp.buckets.end());
    sp.m_max = 256;
    sp.n_max = 512;
    return sp;
}

std::pair<int, int> bucket_shape(int m, int n, const ShapeSpace& space) {
    if (m > space.m_max || n > space.n_max)
        throw ShapeOverflow("execution shape (" + std::to_string(m) + "," + std::to_string(n) + ") exceeds (" +
                            std::to_string(space.m_max) + "," + std::to_string(space.n_max) + ")");
    for (const auto& b : space.buckets)
        if (b.first >= m && b.second >= n) return b;
    return {space.m_max, space.n_max};
}

GraphFootprint graph_memory_footprint(const ShapeSpace& s) {
    // one pool shared by every graph (Alg. 2 lines 2-7); the reference formula,
    // including its LSE pool of W*N*H_s elements (routing.cpp:121-125)
    GraphFootprint fp;
    fp.graph_count = static_cast<std::int64_t>(s.buckets.size());
    const std::int64_t w = s.world_size, hn = s.num_heads, hs = s.head_size, mm = s.m_max, nn = s.n_max;
    const std::int64_t payload = (w * mm + w * nn) * hn * hs + w * nn * hs + mm * static_cast<std::int64_t>(s.hidden_dim);
    const std::int64_t index = mm * static_cast<std::int64_t>(s.max_blocks) + mm;
    fp.buffer_bytes = payload * s.element_size + index * s.index_size;
    return fp;
}

}  // namespace dcpsim
