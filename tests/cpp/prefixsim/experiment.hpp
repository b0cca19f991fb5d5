// TEST-ONLY shim: the reference's paper-figure harness and canned experiments
// (reference experiment.hpp :22-180: mixed_batch_latency_curves,
// grouped_vs_mixed_tpot, short95 / homogeneous / starvation experiments).
// They are not on the decode path, so the product header
// (paper_2605_23389_b200/include/prefixsim/experiment.hpp) leaves them out;
// tests/test_reference_suite.py puts this directory first on the include path
// so the reference's acceptance.cpp and test_cluster_sim.cpp compile unchanged.
#pragma once

#include_next <prefixsim/experiment.hpp>

namespace prefixsim {


struct MixedBatchCurves {
    std::vector<int> long_counts{0, 1, 2, 4};
    std::vector<std::int64_t> generated;
    std::vector<std::vector<double>> latency_ms;
};

// batch 64 of 32-token prompts with 0/1/2/4 replaced by 4096-token prompts
inline MixedBatchCurves mixed_batch_latency_curves(const CalibratedCostModel& model, std::int64_t max_generated = 700,
                                                   std::int64_t step = 20) {
    MixedBatchCurves c;
    c.latency_ms.resize(c.long_counts.size());
    for (std::int64_t g = 0; g <= max_generated; g += step) {
        c.generated.push_back(g);
        for (std::size_t i = 0; i < c.long_counts.size(); ++i) {
            const auto longs = static_cast<std::size_t>(c.long_counts[i]);
            std::vector<std::int64_t> lens(64 - longs, 32 + g);
            lens.resize(64, 4096 + g);
            c.latency_ms[i].push_back(iteration_latency(lens, model).total_ms);
        }
    }
    return c;
}

struct GroupedBatchResult {
    std::vector<std::int64_t> group_lengths;
    std::vector<double> per_group_tpot_ms;
    double grouped_mean_tpot_ms = 0.0;
    double mixed_mean_tpot_ms = 0.0;
    double ratio = 0.0;
};

// 64 length groups (10, 70, ..., 3790): each group batched alone vs one of
// every group per batch, same tokens decoded.
inline GroupedBatchResult grouped_vs_mixed_tpot(const CalibratedCostModel& model, std::int64_t output_len = 32) {
    GroupedBatchResult res;
    for (int g = 0; g < 64; ++g) res.group_lengths.push_back(10 + 60 * g);
    double grouped = 0.0;
    for (const std::int64_t len : res.group_lengths) {
        double sum = 0.0;
        for (std::int64_t k = 0; k < output_len; ++k) {
            const std::vector<std::int64_t> lens(64, len + k);
            sum += iteration_latency(lens, model).total_ms;
        }
        const double tpot = sum / static_cast<double>(output_len);
        res.per_group_tpot_ms.push_back(tpot);
        grouped += tpot;
    }
    res.grouped_mean_tpot_ms = grouped / 64.0;
    double mixed = 0.0;
    for (std::int64_t k = 0; k < output_len; ++k) {
        std::vector<std::int64_t> lens;
        lens.reserve(64);
        for (const std::int64_t len : res.group_lengths) lens.push_back(len + k);
        mixed += iteration_latency(lens, model).total_ms;
    }
    res.mixed_mean_tpot_ms = mixed / static_cast<double>(output_len);
    res.ratio = res.mixed_mean_tpot_ms / res.grouped_mean_tpot_ms;
    return res;
}

inline ExperimentConfig short95_experiment(std::uint64_t seed = 1, Policy policy = Policy::kAligned,
                                           std::int64_t count = 400) {
    ExperimentConfig cfg;
    cfg.model = ModelSpec{4096, 32, 2};
    cfg.sim.policy = policy;
    cfg.sim.seed = seed;
    cfg.sim.cluster.decode_hbm_blocks = 10240;
    cfg.sim.cluster.prefill_hbm_blocks = 10240;
    cfg.sim.constraints.starvation_threshold_ms = 6000;
    WorkloadSpec& w = cfg.workload;
    w.kind = WorkloadSpec::Kind::kSynthetic;
    w.count = count;
    w.short_ratio = 0.95;
    w.short_len_min = 512;
    w.short_len_max = 999;
    w.long_len_min = 1000;
    w.long_len_max = 8000;
    w.output_len.family = OutputLenDist::Family::kUniform;
    w.output_len.lo = 60;
    w.output_len.hi = 68;
    w.arrival.kind = ArrivalProcess::Kind::kPoisson;
    w.arrival.rate_per_s = 400;
    w.seed = seed;
    return cfg;
}

inline ExperimentConfig homogeneous_experiment(std::uint64_t seed = 1) {
    ExperimentConfig cfg;
    cfg.model = ModelSpec{4096, 32, 2};
    cfg.sim.policy = Policy::kAligned;
    cfg.sim.seed = seed;
    WorkloadSpec& w = cfg.workload;
    w.count = 200;
    w.short_ratio = 1.0;
    w.short_len_min = 512;
    w.short_len_max = 512;
    w.output_len.family = OutputLenDist::Family::kFixed;
    w.output_len.fixed_value = 128;
    w.arrival.kind = ArrivalProcess::Kind::kBurst;
    w.seed = seed;
    return cfg;
}

// 300 near-equal prompts around 600 tokens plus one isolated 5000-token prompt
inline std::vector<Request> starvation_workload() {
    std::vector<Request> reqs;
    Rng rng(97);
    double t = 0.0;
    for (int i = 0; i < 300; ++i) {
        Request r;
        r.id = static_cast<RequestId>(reqs.size());
        t += rng.exponential(1000.0 / 150.0);
        r.arrival_ms = t;
        r.prompt_len = 592 + rng.uniform_int(0, 15);
        r.target_output_len = 32;
        reqs.push_back(r);
    }
    Request lone;
    lone.id = static_cast<RequestId>(reqs.size());
    lone.arrival_ms = 100.0;
    lone.prompt_len = 5000;
    lone.target_output_len = 32;
    reqs.push_back(lone);
    return reqs;
}

inline ExperimentConfig starvation_experiment() {
    ExperimentConfig cfg;
    cfg.model = ModelSpec{4096, 32, 2};
    cfg.sim.policy = Policy::kAligned;
    cfg.sim.seed = 97;
    cfg.sim.constraints.starvation_threshold_ms = 500.0;
    cfg.workload.count = 0;
    return cfg;
}

}  // namespace prefixsim
