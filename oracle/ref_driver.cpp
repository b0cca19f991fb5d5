// TEST INFRASTRUCTURE ONLY — thin C driver over the UNMODIFIED reference
// decision path (prefixsim headers under /root/reference/proj/include,
// compiled where they lie by oracle/Makefile into oracle/_ref/).  Used by
// tests/ as the bit-exact oracle for batch composition/order, transfer bytes
// and logs, and by bench.py --impl reference as the reference CPU path.
// Nothing in the product (paper_2605_23389_b200/) links or loads it.
#include <prefixsim/batch_gen.hpp>
#include <prefixsim/experiment.hpp>
#include <prefixsim/io.hpp>

#include "reference_dfs.hpp"  // the reference's own independent DFS oracle (proj/tests)

#include <chrono>
#include <cstdlib>
#include <cstring>
#include <string>

namespace {
thread_local std::string g_err;

char* dup(const std::string& s, long long* len) {
    char* p = static_cast<char*>(std::malloc(s.size() + 1));
    std::memcpy(p, s.data(), s.size());
    p[s.size()] = '\0';
    if (len) *len = static_cast<long long>(s.size());
    return p;
}

template <typename F>
int guard(F&& f) {
    try {
        return f();
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_free(void* p) { std::free(p); }

// experiment_from_json -> run_experiment -> log_to_jsonl (what `prefixsim run` does,
// prefixsim_main.cpp:66-111).  *seconds = wall time of run_experiment alone,
// *iterations = decode iterations simulated.
int ref_run_config_jsonl(const char* config_json, const char* policy, char** out, long long* out_len,
                         double* seconds, long long* iterations) {
    return guard([&] {
        auto cfg = prefixsim::experiment_from_json(prefixsim::json::parse(config_json));
        if (policy) cfg.sim.policy = prefixsim::policy_from_string(policy);
        const auto t0 = std::chrono::steady_clock::now();
        const auto r = prefixsim::run_experiment(cfg);
        const auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        if (iterations) *iterations = static_cast<long long>(r.log.iterations.size());
        *out = dup(prefixsim::log_to_jsonl(r.log), out_len);
        return 0;
    });
}

// Same log, but *seconds times the decision engine alone (Simulation::run over the
// trace, cluster_sim.hpp:773-777): the cost-model calibration and the trace ingest
// happen before the clock starts.
int ref_run_config_timed(const char* config_json, const char* policy, char** out, long long* out_len,
                         double* seconds, long long* iterations) {
    return guard([&] {
        auto cfg = prefixsim::experiment_from_json(prefixsim::json::parse(config_json));
        if (policy) cfg.sim.policy = prefixsim::policy_from_string(policy);
        const prefixsim::CalibratedCostModel model =
            cfg.has_calibration ? cfg.calibration
                                : prefixsim::calibrate(prefixsim::reference_mixed_batch_anchors(), cfg.model).model;
        std::vector<prefixsim::Request> reqs =
            cfg.workload.kind == prefixsim::WorkloadSpec::Kind::kTrace
                ? prefixsim::ingest_trace(cfg.workload.trace_path, cfg.workload.trace_format).requests
                : prefixsim::generate_synthetic(cfg.workload);
        const auto t0 = std::chrono::steady_clock::now();
        const prefixsim::MetricsLog log = prefixsim::run(cfg.sim, std::move(reqs), model);
        const auto t1 = std::chrono::steady_clock::now();
        if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
        if (iterations) *iterations = static_cast<long long>(log.iterations.size());
        *out = dup(prefixsim::log_to_jsonl(log), out_len);
        return 0;
    });
}

// density_first_search on a pool snapshot (all inserted at t = 0, no starvation)
int ref_dfs_batch(const long long* res, long long n, long long b_max, long long k_min, long long* ids,
                  long long* n_out, long long* total_blocks) {
    return guard([&] {
        prefixsim::QuadTree tree;
        for (long long i = 0; i < n; ++i) tree.insert({res[3 * i], res[3 * i + 1], res[3 * i + 2]}, 0.0);
        prefixsim::BatchConstraints c;
        c.b_max = b_max;
        c.k_min = k_min;
        c.starvation_threshold_ms = 1e18;
        const auto b = prefixsim::density_first_search(tree, c, 0.0);
        *n_out = 0;
        *total_blocks = 0;
        if (b) {
            for (const auto& m : b->members) ids[(*n_out)++] = m.id;
            *total_blocks = b->total_blocks;
        }
        return 0;
    });
}

// the reference's independent flat-list DFS oracle (proj/tests/reference_dfs.hpp)
int ref_dfs_flat_oracle(const long long* res, long long n, long long b_max, long long k_min, long long* ids,
                        long long* n_out, long long* total_blocks) {
    return guard([&] {
        std::vector<refdfs::RefRequest> flat;
        for (long long i = 0; i < n; ++i) flat.push_back({res[3 * i], res[3 * i + 1], res[3 * i + 2], i});
        const auto r = refdfs::reference_dfs(flat, b_max, k_min);
        *n_out = 0;
        *total_blocks = 0;
        if (r) {
            for (auto id : r->ids) ids[(*n_out)++] = id;
            *total_blocks = r->total_blocks;
        }
        return 0;
    });
}

// microbenchmark of one reference decision call, ns per call
double ref_time_dfs_ns(const long long* res, long long n, long long b_max, long long k_min, int reps) {
    prefixsim::QuadTree tree;
    for (long long i = 0; i < n; ++i) tree.insert({res[3 * i], res[3 * i + 1], res[3 * i + 2]}, 0.0);
    prefixsim::BatchConstraints c;
    c.b_max = b_max;
    c.k_min = k_min;
    c.starvation_threshold_ms = 1e18;
    long long sink = 0;
    const auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; ++i) {
        const auto b = prefixsim::density_first_search(tree, c, 0.0, 0, false);
        sink += b ? static_cast<long long>(b->members.size()) : 0;
    }
    const auto t1 = std::chrono::steady_clock::now();
    if (sink < 0) return -1;
    return std::chrono::duration<double, std::nano>(t1 - t0).count() / reps;
}

}  // extern "C"
