// SPDX-License-Identifier: Apache-2.0
//
// A reference-API caller: uses only include/dcpsim/*.hpp (the same names and
// signatures as /root/reference/proj/include/dcpsim) and links
// libdcp_b200.so, proving that existing callers relink unchanged.  Replays a
// planner script from stdin and prints results in the format
// tests/test_dropin_gpu.py rebuilds from the oracle.
//
//   cluster NODES IPN PAGE CAP
//   policy KIND HOL UDEG NB [LEN DEG]*     (KIND 0 dcp, 1 least_batch, 2 least_cache, 3 uniform)
//   enqueue ID LEN | step | finish ID | append ID | rebalance | end
#include <deque>
#include <iostream>
#include <limits>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "dcpsim/page_table.hpp"
#include "dcpsim/routing.hpp"
#include "dcpsim/scheduler.hpp"

using namespace dcpsim;

static std::string join(const std::vector<long long>& v) {
    std::string s;
    for (size_t i = 0; i < v.size(); ++i) s += (i ? "," : "") + std::to_string(v[i]);
    return s;
}

int main() {
    std::string cmd;
    int nodes = 1, ipn = 1;
    long long page = 16, cap = 16;
    SchedulerPolicy pol;
    ClusterState cluster;
    bool have_cluster = false;
    std::vector<Request> reqs;
    reqs.reserve(1 << 16);
    std::deque<std::size_t> waiting;
    std::vector<long long> enq;
    std::unique_ptr<Scheduler> sched;
    auto find = [&](long long id) -> Request* {
        for (auto& r : reqs)
            if (r.id == id) return &r;
        return nullptr;
    };
    while (std::cin >> cmd) {
        if (cmd == "cluster") {
            std::cin >> nodes >> ipn >> page >> cap;
            ClusterTopology t;
            t.nodes = nodes;
            t.instances_per_node = ipn;
            t.page_size = page;
            cluster = make_cluster(t, cap);
            have_cluster = true;
        } else if (cmd == "policy") {
            int kind, hol, udeg, nb;
            std::cin >> kind >> hol >> udeg >> nb;
            pol.kind = static_cast<PolicyKind>(kind);
            pol.hol_strict = hol != 0;
            pol.uniform_degree = udeg;
            if (nb > 0) {
                pol.bucket.entries.clear();
                for (int i = 0; i < nb; ++i) {
                    long long len;
                    int deg;
                    std::cin >> len >> deg;
                    pol.bucket.entries.push_back({len, deg});
                }
            }
            pol.validate(cluster.topo);
            sched = std::make_unique<Scheduler>(pol);
        } else if (cmd == "enqueue") {
            long long id, len;
            std::cin >> id >> len;
            Request r;
            r.id = id;
            r.seq_len = len;
            reqs.push_back(r);
            waiting.push_back(reqs.size() - 1);
            enq.push_back(id);
        } else if (cmd == "step") {
            std::vector<std::size_t> active;
            for (std::size_t i = 0; i < reqs.size(); ++i)
                if (reqs[i].state == RequestState::Active) active.push_back(i);
            StepResult res = sched->step(waiting, reqs, active, cluster);
            std::cout << "step c=" << join({res.committed.begin(), res.committed.end()})
                      << " d=" << join({res.deferred.begin(), res.deferred.end()})
                      << " u=" << join({res.unschedulable.begin(), res.unschedulable.end()})
                      << " hol=" << res.hol_events << "\n";
        } else if (cmd == "finish") {
            long long id;
            std::cin >> id;
            int rc = 0;
            try {
                pt_free(id, cluster);
                if (auto* r = find(id)) r->state = RequestState::Finished;
            } catch (const UnknownRequest&) {
                rc = -2;
            }
            std::cout << "finish " << rc << "\n";
        } else if (cmd == "append") {
            long long id;
            std::cin >> id;
            int rc = 0, inst = 0;
            try {
                Request* r = find(id);
                if (!r || !r->placement) throw UnknownRequest("no placement");
                inst = cluster.page_table.append_token(id, *r->placement, cluster.instances);
            } catch (const UnknownRequest&) {
                rc = -2;
                inst = 0;
            }
            std::cout << "append " << rc << " " << inst << "\n";
        } else if (cmd == "rebalance") {
            std::vector<Request*> act;
            for (auto& r : reqs)
                if (r.state == RequestState::Active) act.push_back(&r);
            rebalance_active(act, cluster);
            std::vector<long long> order;
            for (auto* r : act) order.push_back(r->id);
            std::cout << "rebalance " << join(order) << "\n";
        } else if (cmd == "end") {
            break;
        }
    }
    if (!have_cluster) return 1;
    std::vector<long long> kv, b, sc, fr;
    for (const auto& s : cluster.instances) {
        kv.push_back(s.kv_load);
        b.push_back(s.moe_batch);
        sc.push_back(s.shard_count);
        fr.push_back(static_cast<long long>(s.free_frames.size()));
    }
    std::cout << "instances kv=" << join(kv) << " b=" << join(b) << " sc=" << join(sc) << " free=" << join(fr) << "\n";
    for (long long id : enq) {
        Request* r = find(id);
        if (!r || !r->placement) {
            std::cout << "placement " << id << " none\n";
            continue;
        }
        const auto& p = *r->placement;
        std::cout << "placement " << id << " " << join({p.kv_binding.begin(), p.kv_binding.end()}) << " "
                  << join({p.split.begin(), p.split.end()}) << " " << p.moe_binding << "\n";
    }
    cluster.page_table.dump_csv(std::cout);
    std::vector<const Request*> act;
    for (auto& r : reqs)
        if (r.state == RequestState::Active) act.push_back(&r);
    auto cfg = build_binding_config(act, cluster.topo.world_size());
    auto rt = derive_routing_tables(cfg);
    dump_routing_csv(rt, std::cout);
    return 0;
}
