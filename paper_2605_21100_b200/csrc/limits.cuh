// SPDX-License-Identifier: Apache-2.0
#pragma once
namespace dcp {
constexpr int PL_MAXW = 32;  // instances per cluster (one warp lane each)
constexpr int PL_MAXK = 16;  // max CP degree (instances per node)
}  // namespace dcp
