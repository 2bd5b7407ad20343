// SPDX-License-Identifier: Apache-2.0
//
// Two UniformCP Schedulers (and a LeastBatch one) interleaved on ONE cluster,
// written against the dcpsim headers only.  The UniformCP round-robin state is
// per Scheduler (reference scheduler.hpp:88, scheduler.cpp:189-222), so the
// MoE bindings below depend on which Scheduler admitted what.  The same source
// compiled against the reference (tools/make_golden.py, -Ddcpsim=dcpsim_ref)
// produced tests/golden/two_schedulers.txt; the drop-in must print it exactly.
#include <deque>
#include <iostream>
#include <vector>

#include "dcpsim/page_table.hpp"
#include "dcpsim/scheduler.hpp"

using namespace dcpsim;

int main() {
    ClusterTopology topo;
    topo.nodes = 1;
    topo.instances_per_node = 4;
    auto cluster = make_cluster(topo, 4096);
    SchedulerPolicy u;
    u.kind = PolicyKind::UniformCP;
    u.uniform_degree = 2;
    SchedulerPolicy lb;
    lb.kind = PolicyKind::LeastBatch;
    Scheduler s1(u), s2(u), s3(lb);
    Scheduler* order[] = {&s1, &s1, &s2, &s3, &s1, &s2, &s2, &s1, &s3, &s2, &s1, &s1};
    std::vector<Request> reqs;
    reqs.reserve(64);
    std::vector<std::size_t> active;
    int next = 0;
    for (int round = 0; round < 12; ++round) {
        std::deque<std::size_t> waiting;
        for (int j = 0; j < 2; ++j) {
            Request r;
            r.id = 100 + next;
            r.seq_len = 37 + 211 * next;
            reqs.push_back(r);
            waiting.push_back(reqs.size() - 1);
            ++next;
        }
        auto res = order[round]->step(waiting, reqs, active, cluster);
        std::cout << "round " << round;
        for (auto id : res.committed) {
            const Request& r = reqs[static_cast<std::size_t>(id - 100)];
            std::cout << " " << id << ":" << r.placement->moe_binding << "/";
            for (auto s : r.placement->kv_binding) std::cout << s;
            active.push_back(static_cast<std::size_t>(id - 100));
        }
        std::cout << " B";
        for (const auto& in : cluster.instances) std::cout << " " << in.moe_batch;
        std::cout << "\n";
    }
    return 0;
}
