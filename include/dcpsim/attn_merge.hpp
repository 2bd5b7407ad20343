// SPDX-License-Identifier: Apache-2.0
//
// dcpsim drop-in: partial attention and LSE merge (reference
// attn_merge.hpp:17-121).  The reference defines these as header templates
// running on the host; here they are declared for T in {float, double} and
// executed on the device (K1f / K9f, csrc/attn_contig.cuh) — the host spans
// are copied in, the results copied out.  The bf16 paged decode path used by
// the data plane is dcp_splitkv_decode_attn (K1).
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

extern template std::vector<float> reference_attention<float>(std::span<const float>, std::span<const float>,
                                                              std::span<const float>, std::int64_t, int, float);
extern template std::vector<double> reference_attention<double>(std::span<const double>, std::span<const double>,
                                                                std::span<const double>, std::int64_t, int, double);
extern template AttnShardResult<float> shard_attention<float>(std::span<const float>, std::span<const float>,
                                                              std::span<const float>, std::int64_t, int, float);
extern template AttnShardResult<double> shard_attention<double>(std::span<const double>, std::span<const double>,
                                                                std::span<const double>, std::int64_t, int, double);
extern template std::vector<float> lse_merge<float>(std::span<const AttnShardResult<float>>);
extern template std::vector<double> lse_merge<double>(std::span<const AttnShardResult<double>>);
extern template std::vector<AttnShardResult<float>> partitioned_shard_attention<float>(
    std::span<const float>, std::span<const float>, std::span<const float>, int, float, std::span<const std::int64_t>);
extern template std::vector<AttnShardResult<double>> partitioned_shard_attention<double>(
    std::span<const double>, std::span<const double>, std::span<const double>, int, double,
    std::span<const std::int64_t>);

}  // namespace dcpsim

#pragma GCC visibility pop
