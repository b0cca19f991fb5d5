// CPU test of the per-pair orchestrator's data-plane interface (include/prefixsim/cluster_sim.hpp):
//   1. a recording DataPlane sees exactly the log's transfers (route, request, bytes, link, sync), the
//      batch prefetch members in page-table order, every release, and every iteration's running set
//      whose prefix lengths equal the record's;
//   2. wall-clock mode: a plane reporting a fixed measured duration per step drives the clock — the
//      log's iteration times are the measured ones and the run stays valid (census, completion).
// usage: orchestrator_test <config.json> <policy>
#include <prefixsim/experiment.hpp>
#include <prefixsim/io.hpp>

#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <map>
#include <sstream>
#include <string>

using namespace prefixsim;

#define CHECK(c)                                                                  \
    do {                                                                          \
        if (!(c)) {                                                               \
            std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #c);  \
            std::exit(1);                                                         \
        }                                                                         \
    } while (0)

struct Recorder : DataPlane {
    std::vector<KvMove> moves;
    std::vector<std::vector<RequestId>> batches;
    std::vector<RequestId> released_ids;
    std::int64_t steps = 0, in_place = 0;
    double measured = -1.0;  // >= 0: wall-clock mode with this step time
    void kv_move(const KvMove& m) override {
        moves.push_back(m);
        if (m.route == KvRoute::kBatchPrefetch) {
            CHECK(m.members != nullptr && !m.members->empty() && m.request == -1);
            batches.push_back(*m.members);
        } else {
            CHECK(m.members == nullptr && m.request >= 0);
        }
    }
    void released(RequestId id) override { released_ids.push_back(id); }
    void prompt_in_place(RequestId, std::int64_t blocks) override {
        CHECK(blocks > 0);
        ++in_place;
    }
    void decode_step(const IterationRecord& rec, const std::vector<RunningMember>& running) override {
        CHECK(running.size() == rec.prefix_lengths.size());
        for (std::size_t i = 0; i < running.size(); ++i) CHECK(running[i].prefix_len == rec.prefix_lengths[i]);
        ++steps;
    }
    bool measured_step_ms(const IterationRecord&, double* ms) override {
        if (measured < 0) return false;
        *ms = measured;
        return true;
    }
};

int main(int argc, char** argv) {
    if (argc < 3) return 2;
    std::ifstream f(argv[1]);
    std::stringstream ss;
    ss << f.rdbuf();
    ExperimentConfig cfg = experiment_from_json(json::parse(ss.str()));
    cfg.sim.policy = policy_from_string(argv[2]);
    const CalibratedCostModel model =
        cfg.has_calibration ? cfg.calibration : calibrate(reference_mixed_batch_anchors(), cfg.model).model;
    const std::vector<Request> reqs = generate_synthetic(cfg.workload);

    // 1. orders == log
    {
        PairOrchestrator engine(cfg.sim, model, reqs);
        Recorder plane;
        engine.attach(&plane);
        const MetricsLog log = engine.run();
        CHECK(plane.moves.size() == log.transfers.size());
        for (std::size_t i = 0; i < log.transfers.size(); ++i) {
            const TransferRecord& t = log.transfers[i];
            const KvMove& m = plane.moves[i];
            CHECK(t.kind == route_name(m.route) && t.bytes == m.bytes && t.link == m.link &&
                  t.synchronous == m.synchronous && t.request_id == m.request && t.duration_ms == m.duration_ms);
        }
        std::size_t b = 0, r = 0;
        for (const ActionRecord& a : log.actions) {
            if (a.action == "release") CHECK(plane.released_ids.at(r++) == a.request_id);
        }
        CHECK(r == plane.released_ids.size());
        std::vector<RequestId> batched;
        for (const ActionRecord& a : log.actions)
            if (a.action == "batch") batched.push_back(a.request_id);
        std::vector<RequestId> flat;
        for (const auto& v : plane.batches) flat.insert(flat.end(), v.begin(), v.end());
        CHECK(flat == batched);
        (void)b;
        CHECK(plane.steps == static_cast<std::int64_t>(log.iterations.size()) && plane.steps > 0);
        // the same decisions as the plain run() (a plane never changes them)
        CHECK(log_to_jsonl(log) == log_to_jsonl(run(cfg.sim, reqs, model)));
        std::printf("orders: %zu moves, %zu batches, %zu releases, %lld steps, %lld in-place prompts\n",
                    plane.moves.size(), plane.batches.size(), plane.released_ids.size(),
                    static_cast<long long>(plane.steps), static_cast<long long>(plane.in_place));
    }
    // 2. wall clock
    {
        PairOrchestrator engine(cfg.sim, model, reqs);
        Recorder plane;
        plane.measured = 0.75;
        engine.attach(&plane);
        const MetricsLog log = engine.run();  // validate_invariants: census + token conservation inside
        CHECK(!log.iterations.empty());
        for (const IterationRecord& it : log.iterations) {
            CHECK(it.compute_ms == 0.75);
            CHECK(it.end_ms == it.start_ms + 0.75);
        }
        std::size_t done = 0;
        for (const RequestRecord& rr : log.requests) done += (!rr.rejected && rr.completed_ms >= 0) ? 1 : 0;
        CHECK(done > 0);
        std::printf("wall clock: %zu iterations at 0.75 ms, %zu requests completed, tok/s %.1f\n",
                    log.iterations.size(), done, decode_throughput(log));
    }
    std::printf("PASS\n");
    return 0;
}
