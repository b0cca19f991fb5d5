// C ABI of the host-side decision path (include/asv.h): the reference-API
// engine in virtual-clock mode and the density-first-search batcher.  The C++
// exceptions of the reference API map to ASV_ERR_* codes with the same
// messages (invalid_argument -> ASV_ERR_INVALID, logic_error -> ASV_ERR_LOGIC,
// runtime_error and the rest -> ASV_ERR_RUNTIME).
#include <prefixsim/batch_gen.hpp>
#include <prefixsim/experiment.hpp>
#include <prefixsim/io.hpp>

#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>

#include "../../include/asv.h"
#include "asv_internal.h"
#include "engine_internal.h"

namespace asv {

template <typename F>
int guarded(F&& fn) {
    try {
        return fn();
    } catch (const std::invalid_argument& e) {
        return fail(ASV_ERR_INVALID, e.what());
    } catch (const std::logic_error& e) {
        return fail(ASV_ERR_LOGIC, e.what());
    } catch (const std::exception& e) {
        return fail(ASV_ERR_RUNTIME, e.what());
    }
}

char* dup_string(const std::string& s, int64_t* len) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    if (p == nullptr) throw std::runtime_error("out of host memory");
    std::memcpy(p, s.data(), s.size());
    p[s.size()] = '\0';
    if (len) *len = static_cast<int64_t>(s.size());
    return p;
}

std::vector<prefixsim::Request> load_workload(const prefixsim::ExperimentConfig& cfg) {
    return cfg.workload.kind == prefixsim::WorkloadSpec::Kind::kTrace
               ? prefixsim::ingest_trace(cfg.workload.trace_path, cfg.workload.trace_format).requests
               : prefixsim::generate_synthetic(cfg.workload);
}

// Data-parallel shard of a trace: request i goes to shard i % count (arrival
// times and order preserved; PairOrchestrator::run re-numbers ids to local indices,
// cluster_sim.hpp:137-139, so global id = local * count + index).
void shard_requests(std::vector<prefixsim::Request>& reqs, int32_t index, int32_t count) {
    if (count < 1 || index < 0 || index >= count) throw std::invalid_argument("bad shard index/count");
    if (count == 1) return;
    std::vector<prefixsim::Request> mine;
    for (std::size_t i = static_cast<std::size_t>(index); i < reqs.size(); i += static_cast<std::size_t>(count)) {
        mine.push_back(reqs[i]);
    }
    reqs.swap(mine);
}

}  // namespace asv

using namespace asv;

extern "C" {

int asv_run_config_jsonl(const char* config_json, const char* policy_override, char** out, int64_t* out_len) {
    return guarded([&] {
        if (config_json == nullptr || out == nullptr) throw std::invalid_argument("null config/out");
        prefixsim::ExperimentConfig cfg = prefixsim::experiment_from_json(prefixsim::json::parse(config_json));
        if (policy_override != nullptr) cfg.sim.policy = prefixsim::policy_from_string(policy_override);
        const prefixsim::ExperimentResult r = prefixsim::run_experiment(cfg);
        *out = dup_string(prefixsim::log_to_jsonl(r.log), out_len);
        return ASV_OK;
    });
}

int asv_run_config_jsonl_shard(const char* config_json, const char* policy_override, int32_t shard_index,
                               int32_t shard_count, char** out, int64_t* out_len) {
    return guarded([&] {
        if (config_json == nullptr || out == nullptr) throw std::invalid_argument("null config/out");
        prefixsim::ExperimentConfig cfg = prefixsim::experiment_from_json(prefixsim::json::parse(config_json));
        if (policy_override != nullptr) cfg.sim.policy = prefixsim::policy_from_string(policy_override);
        std::vector<prefixsim::Request> reqs = load_workload(cfg);
        shard_requests(reqs, shard_index, shard_count);
        const prefixsim::CalibratedCostModel model =
            cfg.has_calibration ? cfg.calibration
                                : prefixsim::calibrate(prefixsim::reference_mixed_batch_anchors(), cfg.model).model;
        const prefixsim::MetricsLog log = prefixsim::run(cfg.sim, std::move(reqs), model);
        *out = dup_string(prefixsim::log_to_jsonl(log), out_len);
        return ASV_OK;
    });
}

int asv_dfs_batch(const int64_t* residents, int64_t n, int64_t b_max, int64_t k_min, int64_t* ids_out,
                  int64_t* n_out, int64_t* total_blocks_out) {
    return guarded([&] {
        prefixsim::QuadTree tree;
        for (int64_t i = 0; i < n; ++i) {
            tree.insert({residents[3 * i], residents[3 * i + 1], residents[3 * i + 2]}, 0.0);
        }
        prefixsim::BatchConstraints c;
        c.b_max = b_max;
        c.k_min = k_min;
        c.starvation_threshold_ms = 1e18;
        const auto batch = prefixsim::density_first_search(tree, c, 0.0);
        *n_out = 0;
        *total_blocks_out = 0;
        if (batch) {
            for (const auto& m : batch->members) ids_out[(*n_out)++] = m.id;
            *total_blocks_out = batch->total_blocks;
        }
        return ASV_OK;
    });
}

}  // extern "C"
