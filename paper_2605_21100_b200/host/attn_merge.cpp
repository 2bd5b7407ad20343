// SPDX-License-Identifier: Apache-2.0
//
// dcpsim drop-in: shard_attention / reference_attention / lse_merge /
// sharded_attention_merge on the device (K1f / K9f, csrc/attn_contig.cuh).
// Host spans are staged into a grow-only device scratch buffer; the kernel
// results are copied back into the reference's return types.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <limits>

#include "dcpsim/attn_merge.hpp"
#include "dcpsim/device.hpp"

namespace dcpsim {

namespace {

struct Scratch {
    void* p = nullptr;
    size_t bytes = 0;
    ~Scratch() {
        if (p) cudaFree(p);
    }
    char* get(size_t n) {
        if (n > bytes) {
            if (p) cudaFree(p);
            if (cudaMalloc(&p, n) != cudaSuccess) throw SimError("cudaMalloc failed for attention scratch");
            bytes = n;
        }
        return static_cast<char*>(p);
    }
};
thread_local Scratch g_scratch;

size_t al(size_t x) { return (x + 255) & ~size_t(255); }

void h2d(void* dst, const void* src, size_t n) {
    if (n && cudaMemcpy(dst, src, n, cudaMemcpyHostToDevice) != cudaSuccess) throw SimError("H2D copy failed");
}
void d2h(void* dst, const void* src, size_t n) {
    if (n && cudaMemcpy(dst, src, n, cudaMemcpyDeviceToHost) != cudaSuccess) throw SimError("D2H copy failed");
}

// Partial attention for `items` shards of one query over contiguous K/V.
template <typename T>
void run_items(std::span<const T> q, std::span<const T> keys, std::span<const T> values, int d, T scale,
               const std::vector<std::int64_t>& starts, const std::vector<std::int64_t>& lens, std::vector<T>& outs,
               std::vector<T>& lses) {
    dcp_ctx* ctx = device::context();
    const int n = static_cast<int>(starts.size());
    std::int64_t kv_elems = 0;
    for (int i = 0; i < n; ++i) kv_elems = std::max(kv_elems, (starts[i] + lens[i]) * d);
    const size_t bq = al(sizeof(T) * d), bkv = al(sizeof(T) * std::max<std::int64_t>(kv_elems, 1)),
                 bo = al(sizeof(T) * d * n), bl = al(sizeof(T) * n), bi = al(sizeof(std::int64_t) * n);
    char* base = g_scratch.get(bq + 2 * bkv + bo + bl + 3 * bi);
    T* dq = reinterpret_cast<T*>(base);
    T* dk = reinterpret_cast<T*>(base + bq);
    T* dv = reinterpret_cast<T*>(base + bq + bkv);
    T* dout = reinterpret_cast<T*>(base + bq + 2 * bkv);
    T* dlse = reinterpret_cast<T*>(base + bq + 2 * bkv + bo);
    auto* qoff = reinterpret_cast<std::int64_t*>(base + bq + 2 * bkv + bo + bl);
    auto* kvoff = qoff + bi / sizeof(std::int64_t);
    auto* dlen = kvoff + bi / sizeof(std::int64_t);
    std::vector<std::int64_t> qo(n, 0), ko(n);
    for (int i = 0; i < n; ++i) ko[i] = starts[i] * d;
    h2d(dq, q.data(), sizeof(T) * d);
    h2d(dk, keys.data(), sizeof(T) * kv_elems);
    h2d(dv, values.data(), sizeof(T) * kv_elems);
    h2d(qoff, qo.data(), 8 * n);
    h2d(kvoff, ko.data(), 8 * n);
    h2d(dlen, lens.data(), 8 * n);
    device::check(dcp_shard_attention_batch(ctx, sizeof(T), n, d, static_cast<double>(scale), dq, dk, dv, qoff,
                                            kvoff, dlen, dout, dlse, nullptr));
    outs.resize(static_cast<size_t>(n) * d);
    lses.resize(n);
    d2h(outs.data(), dout, sizeof(T) * d * n);
    d2h(lses.data(), dlse, sizeof(T) * n);
}

template <typename T>
std::vector<T> merge_device(const std::vector<T>& outs, const std::vector<T>& lses, int d) {
    dcp_ctx* ctx = device::context();
    const int n = static_cast<int>(lses.size());
    const size_t bo = al(sizeof(T) * outs.size()), bl = al(sizeof(T) * n), bm = al(sizeof(T) * d);
    char* base = g_scratch.get(bo + bl + bm + 256);
    T* dout = reinterpret_cast<T*>(base);
    T* dl = reinterpret_cast<T*>(base + bo);
    T* dm = reinterpret_cast<T*>(base + bo + bl);
    auto* off = reinterpret_cast<std::int64_t*>(base + bo + bl + bm);
    const std::int64_t o2[2] = {0, n};
    h2d(dout, outs.data(), sizeof(T) * outs.size());
    h2d(dl, lses.data(), sizeof(T) * n);
    h2d(off, o2, sizeof(o2));
    device::check(dcp_lse_merge_batch(ctx, sizeof(T), 1, d, off, dout, dl, dm, nullptr, nullptr));
    std::vector<T> r(static_cast<size_t>(d));
    d2h(r.data(), dm, sizeof(T) * d);
    return r;
}

}  // namespace

namespace impl {

template <typename T>
AttnShardResult<T> shard_attention_t(std::span<const T> q, std::span<const T> keys, std::span<const T> values,
                                   std::int64_t length, int head_dim, T scale) {
    if (length < 1) throw EmptyShard("shard_attention over zero keys");  // attn_merge.hpp:57
    std::vector<T> outs, lses;
    run_items<T>(q, keys, values, head_dim, scale, {0}, {length}, outs, lses);
    AttnShardResult<T> r;
    r.partial_out = std::move(outs);
    r.lse = lses[0];
    return r;
}

template <typename T>
std::vector<T> reference_attention_t(std::span<const T> q, std::span<const T> keys, std::span<const T> values,
                                   std::int64_t length, int head_dim, T scale) {
    if (length < 1) return std::vector<T>(static_cast<size_t>(head_dim), std::numeric_limits<T>::quiet_NaN());
    return shard_attention_t<T>(q, keys, values, length, head_dim, scale).partial_out;
}

template <typename T>
std::vector<T> lse_merge_t(std::span<const AttnShardResult<T>> partials) {
    if (partials.empty()) throw EmptyShard("lse_merge of zero partials");  // attn_merge.hpp:88
    const int d = static_cast<int>(partials.front().partial_out.size());
    std::vector<T> outs, lses;
    for (const auto& p : partials) {
        outs.insert(outs.end(), p.partial_out.begin(), p.partial_out.end());
        lses.push_back(p.lse);
    }
    return merge_device<T>(outs, lses, d);
}

template <typename T>
std::vector<AttnShardResult<T>> partitioned_shard_attention_t(std::span<const T> q, std::span<const T> keys,
                                                            std::span<const T> values, int head_dim, T scale,
                                                            std::span<const std::int64_t> bounds) {
    // contiguous partition, exclusive ends; zero-width shards receive no query
    // and stay empty (attn_merge.cpp:9-33)
    std::vector<AttnShardResult<T>> res(bounds.size());
    std::vector<std::int64_t> starts, lens, which;
    std::int64_t start = 0;
    for (std::size_t i = 0; i < bounds.size(); ++i) {
        if (bounds[i] > start) {
            starts.push_back(start);
            lens.push_back(bounds[i] - start);
            which.push_back(static_cast<std::int64_t>(i));
        }
        start = bounds[i];
    }
    if (starts.empty()) return res;
    std::vector<T> outs, lses;
    run_items<T>(q, keys, values, head_dim, scale, starts, lens, outs, lses);
    for (std::size_t j = 0; j < which.size(); ++j) {
        auto& r = res[static_cast<std::size_t>(which[j])];
        r.partial_out.assign(outs.begin() + static_cast<long>(j) * head_dim,
                             outs.begin() + static_cast<long>(j + 1) * head_dim);
        r.lse = lses[j];
    }
    return res;
}

}  // namespace impl

#pragma GCC visibility push(default)

namespace {
template <typename T>
std::vector<T> merge_impl(std::span<const T> q, std::span<const T> keys, std::span<const T> values, int d, T scale,
                          std::span<const std::int64_t> bounds) {
    auto parts = impl::partitioned_shard_attention_t<T>(q, keys, values, d, scale, bounds);
    std::vector<AttnShardResult<T>> live;
    for (auto& p : parts)
        if (!p.partial_out.empty()) live.push_back(std::move(p));  // drop empty shards, keep order
    return impl::lse_merge_t<T>(live);
}
}  // namespace

std::vector<float> sharded_attention_merge(std::span<const float> q, std::span<const float> keys,
                                           std::span<const float> values, int head_dim, float scale,
                                           std::span<const std::int64_t> bounds, bool) {
    return merge_impl<float>(q, keys, values, head_dim, scale, bounds);
}

std::vector<double> sharded_attention_merge(std::span<const double> q, std::span<const double> keys,
                                            std::span<const double> values, int head_dim, double scale,
                                            std::span<const std::int64_t> bounds, bool) {
    return merge_impl<double>(q, keys, values, head_dim, scale, bounds);
}

template <>
std::vector<float> reference_attention<float>(std::span<const float> q, std::span<const float> k,
                                              std::span<const float> v, std::int64_t n, int d, float sc) {
    return impl::reference_attention_t<float>(q, k, v, n, d, sc);
}
template <>
std::vector<double> reference_attention<double>(std::span<const double> q, std::span<const double> k,
                                                std::span<const double> v, std::int64_t n, int d, double sc) {
    return impl::reference_attention_t<double>(q, k, v, n, d, sc);
}
template <>
AttnShardResult<float> shard_attention<float>(std::span<const float> q, std::span<const float> k,
                                              std::span<const float> v, std::int64_t n, int d, float sc) {
    return impl::shard_attention_t<float>(q, k, v, n, d, sc);
}
template <>
AttnShardResult<double> shard_attention<double>(std::span<const double> q, std::span<const double> k,
                                                std::span<const double> v, std::int64_t n, int d, double sc) {
    return impl::shard_attention_t<double>(q, k, v, n, d, sc);
}
template <>
std::vector<float> lse_merge<float>(std::span<const AttnShardResult<float>> p) {
    return impl::lse_merge_t<float>(p);
}
template <>
std::vector<double> lse_merge<double>(std::span<const AttnShardResult<double>> p) {
    return impl::lse_merge_t<double>(p);
}
template <>
std::vector<AttnShardResult<float>> partitioned_shard_attention<float>(std::span<const float> q,
                                                                       std::span<const float> k,
                                                                       std::span<const float> v, int d, float sc,
                                                                       std::span<const std::int64_t> b) {
    return impl::partitioned_shard_attention_t<float>(q, k, v, d, sc, b);
}
template <>
std::vector<AttnShardResult<double>> partitioned_shard_attention<double>(std::span<const double> q,
                                                                         std::span<const double> k,
                                                                         std::span<const double> v, int d,
                                                                         double sc, std::span<const std::int64_t> b) {
    return impl::partitioned_shard_attention_t<double>(q, k, v, d, sc, b);
}

#pragma GCC visibility pop

}  // namespace dcpsim
