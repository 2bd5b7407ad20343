// SPDX-License-Identifier: Apache-2.0
//
// dcpsim drop-in: partial attention and LSE merge (reference
// attn_merge.hpp:17-121).  The reference defines these as header templates
// running on the host; here float and double are explicit specializations
// executed on the device (K1f / K9f, csrc/attn_contig.cuh) — the host spans
// are copied in, the results copied out — and any other T goes through the
// double path.  The bf16 paged decode path used by the data plane is
// dcp_splitkv_decode_attn (K1).
#pragma once

#include <cstdint>
#include <span>
#include <vector>

#include "dcpsim/types.hpp"

#pragma GCC visibility push(default)

namespace dcpsim {

template <typename T>
struct AttnShardResult {
    std::vector<T> partial_out;
    T lse = T(0);
};

// Primary templates (any arithmetic T), declared first so the float / double explicit
// specializations below are known before any use.
template <typename T>
std::vector<T> reference_attention(std::span<const T> q, std::span<const T> keys, std::span<const T> values,
                                   std::int64_t length, int head_dim, T scale);

template <typename T>
AttnShardResult<T> shard_attention(std::span<const T> q, std::span<const T> keys, std::span<const T> values,
                                   std::int64_t length, int head_dim, T scale);

template <typename T>
std::vector<T> lse_merge(std::span<const AttnShardResult<T>> partials);

template <typename T>
std::vector<AttnShardResult<T>> partitioned_shard_attention(std::span<const T> q, std::span<const T> keys,
                                                            std::span<const T> values, int head_dim, T scale,
                                                            std::span<const std::int64_t> bounds);

std::vector<float> sharded_attention_merge(std::span<const float> q, std::span<const float> keys,
                                           std::span<const float> values, int head_dim, float scale,
                                           std::span<const std::int64_t> bounds, bool parallel);
std::vector<double> sharded_attention_merge(std::span<const double> q, std::span<const double> keys,
                                            std::span<const double> values, int head_dim, double scale,
                                            std::span<const std::int64_t> bounds, bool parallel);

// float and double: device kernels (K1f / K9f), defined in the library.
template <>
std::vector<float> reference_attention<float>(std::span<const float>, std::span<const float>, std::span<const float>,
                                              std::int64_t, int, float);
template <>
std::vector<double> reference_attention<double>(std::span<const double>, std::span<const double>,
                                                std::span<const double>, std::int64_t, int, double);
template <>
AttnShardResult<float> shard_attention<float>(std::span<const float>, std::span<const float>, std::span<const float>,
                                              std::int64_t, int, float);
template <>
AttnShardResult<double> shard_attention<double>(std::span<const double>, std::span<const double>,
                                                std::span<const double>, std::int64_t, int, double);
template <>
std::vector<float> lse_merge<float>(std::span<const AttnShardResult<float>>);
template <>
std::vector<double> lse_merge<double>(std::span<const AttnShardResult<double>>);
template <>
std::vector<AttnShardResult<float>> partitioned_shard_attention<float>(std::span<const float>, std::span<const float>,
                                                                       std::span<const float>, int, float,
                                                                       std::span<const std::int64_t>);
template <>
std::vector<AttnShardResult<double>> partitioned_shard_attention<double>(std::span<const double>,
                                                                         std::span<const double>,
                                                                         std::span<const double>, int, double,
                                                                         std::span<const std::int64_t>);

// Any other T (the reference's templates accept every floating type, attn_merge.hpp:25-100):
// widened to double, computed by the double device path, narrowed back.
namespace detail {
template <typename T>
std::vector<double> widen(std::span<const T> s) {
    return std::vector<double>(s.begin(), s.end());
}
template <typename T>
std::vector<T> narrow(const std::vector<double>& v) {
    return std::vector<T>(v.begin(), v.end());
}
template <typename T>
AttnShardResult<T> narrow(const AttnShardResult<double>& r) {
    return AttnShardResult<T>{narrow<T>(r.partial_out), static_cast<T>(r.lse)};
}
}  // namespace detail

template <typename T>
std::vector<T> reference_attention(std::span<const T> q, std::span<const T> keys, std::span<const T> values,
                                   std::int64_t length, int head_dim, T scale) {
    const auto qd = detail::widen(q), kd = detail::widen(keys), vd = detail::widen(values);
    return detail::narrow<T>(reference_attention<double>(qd, kd, vd, length, head_dim, static_cast<double>(scale)));
}

template <typename T>
AttnShardResult<T> shard_attention(std::span<const T> q, std::span<const T> keys, std::span<const T> values,
                                   std::int64_t length, int head_dim, T scale) {
    const auto qd = detail::widen(q), kd = detail::widen(keys), vd = detail::widen(values);
    return detail::narrow<T>(shard_attention<double>(qd, kd, vd, length, head_dim, static_cast<double>(scale)));
}

template <typename T>
std::vector<T> lse_merge(std::span<const AttnShardResult<T>> partials) {
    std::vector<AttnShardResult<double>> pd;
    pd.reserve(partials.size());
    for (const auto& p : partials)
        pd.push_back(AttnShardResult<double>{std::vector<double>(p.partial_out.begin(), p.partial_out.end()),
                                             static_cast<double>(p.lse)});
    return detail::narrow<T>(lse_merge<double>(std::span<const AttnShardResult<double>>(pd)));
}

template <typename T>
std::vector<AttnShardResult<T>> partitioned_shard_attention(std::span<const T> q, std::span<const T> keys,
                                                            std::span<const T> values, int head_dim, T scale,
                                                            std::span<const std::int64_t> bounds) {
    const auto qd = detail::widen(q), kd = detail::widen(keys), vd = detail::widen(values);
    const auto rd = partitioned_shard_attention<double>(qd, kd, vd, head_dim, static_cast<double>(scale), bounds);
    std::vector<AttnShardResult<T>> out;
    out.reserve(rd.size());
    for (const auto& r : rd) out.push_back(detail::narrow<T>(r));
    return out;
}

}  // namespace dcpsim

#pragma GCC visibility pop
