// Host-only glue shared by the engine entry points (capi_engine.cpp,
// executor.cpp): trace loading and data-parallel sharding.
#pragma once

#include <prefixsim/io.hpp>

#include <cstdint>
#include <vector>

namespace asv {

std::vector<prefixsim::Request> load_workload(const prefixsim::ExperimentConfig& cfg);
void shard_requests(std::vector<prefixsim::Request>& reqs, int32_t index, int32_t count);

}  // namespace asv
