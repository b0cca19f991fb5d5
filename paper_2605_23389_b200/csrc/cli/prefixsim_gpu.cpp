// prefixsim_gpu: the reference CLI (tools/prefixsim_main.cpp) with the decode
// path executed on a B200.
//
//   run        ~ cmd_run (prefixsim_main.cpp:66-111): same flags, same artefacts
//                (config_used.json, log.jsonl, summary.json, ttft_cdf.csv,
//                sched_cdf.csv; SVG charts omitted) from the same decisions —
//                log.jsonl is byte-identical to the reference's — plus
//                gpu_stats.json with the measured decode tokens/s, attention
//                HBM GB/s and bytes moved.  The engine runs through the C ABI
//                (asv_engine_run_ex, include/asv.h).
//   compare    ~ cmd_compare (:113-160): policy x seed sweep on the virtual clock
//                (the reference's decisions; add --gpu to also execute each run).
//   trace-gen  ~ cmd_trace_gen (:258-284).
//   calibrate  ~ cmd_calibrate (:51-64).
// `paperfig` (figure reproductions, SVG) is not part of the decode hot path.
//
// Host-only C++ above the C ABI; CLI11 is not in this image, so flags are
// parsed here with the reference's names and defaults.
#include <prefixsim/experiment.hpp>
#include <prefixsim/io.hpp>
#include <prefixsim/metrics.hpp>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <filesystem>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "../../../include/asv.h"

namespace {

using prefixsim::json;

struct Args {
    std::map<std::string, std::string> opt;
    std::vector<std::string> flags;
    bool has(const std::string& k) const { return opt.count(k) != 0; }
    bool flag(const std::string& k) const {
        for (const auto& f : flags) {
            if (f == k) return true;
        }
        return false;
    }
    std::string get(const std::string& k, const std::string& d = "") const {
        const auto it = opt.find(k);
        return it == opt.end() ? d : it->second;
    }
    int64_t get_i(const std::string& k, int64_t d) const { return has(k) ? std::stoll(get(k)) : d; }
};

// --key value / --key=value / --flag (flags listed in `boolean`)
Args parse(int argc, char** argv, int first, const std::vector<std::string>& boolean) {
    Args a;
    for (int i = first; i < argc; ++i) {
        std::string k = argv[i];
        if (k.rfind("--", 0) != 0) throw std::invalid_argument("unexpected argument: " + k);
        const auto eq = k.find('=');
        if (eq != std::string::npos) {
            a.opt[k.substr(0, eq)] = k.substr(eq + 1);
            continue;
        }
        bool is_flag = false;
        for (const auto& b : boolean) is_flag = is_flag || b == k;
        if (is_flag) {
            a.flags.push_back(k);
        } else {
            if (i + 1 >= argc) throw std::invalid_argument("missing value for " + k);
            a.opt[k] = argv[++i];
        }
    }
    return a;
}

std::string output_root() {
    if (const char* env = std::getenv("PREFIXSIM_OUTPUT_ROOT")) return env;
    return ".";
}

std::string join_path(const std::string& root, const std::string& leaf) {
    return (std::filesystem::path(root) / leaf).string();
}

// a relative trace path is tried against the working directory (the reference's
// behaviour), then against the config's directory and its parent
void resolve_trace(json& cfg, const std::string& config_path) {
    if (!cfg.contains("workload") || cfg["workload"].value("kind", "") != "trace") return;
    const std::filesystem::path p = cfg["workload"].value("path", "");
    if (p.empty() || p.is_absolute() || std::filesystem::exists(p)) return;
    const std::filesystem::path dir = std::filesystem::absolute(config_path).parent_path();
    for (const auto& base : {dir, dir.parent_path()}) {
        if (std::filesystem::exists(base / p)) {
            cfg["workload"]["path"] = (base / p).string();
            return;
        }
    }
}

// attention shape of the config: the "b200" section if present, else the model
// (hidden_dim / 128 heads of d = 128, num_kv_heads default = heads)
void shape_of(const json& cfg, const Args& a, asv_engine_opts& o) {
    const json m = cfg.value("model", json::object());
    const json b = cfg.value("b200", json::object());
    const int64_t hidden = m.value("hidden_dim", int64_t(4096));
    const int64_t heads = b.value("num_q_heads", m.value("num_heads", hidden / 128));
    o.num_q_heads = static_cast<int32_t>(a.get_i("--heads", heads));
    o.num_kv_heads = static_cast<int32_t>(a.get_i("--kv-heads", b.value("num_kv_heads", m.value("num_kv_heads", heads))));
    o.num_layers = static_cast<int32_t>(a.get_i("--layers", b.value("num_layers", m.value("num_layers", int64_t(32)))));
}

int cmd_run(const Args& a) {
    const std::string config_path = a.get("--config");
    if (config_path.empty()) throw std::invalid_argument("run: --config is required");
    json used = json::parse(prefixsim::read_file(config_path));
    // flag semantics of the reference's cmd_run (prefixsim_main.cpp:70-85)
    if (a.has("--policy")) used["policy"] = a.get("--policy");
    if (a.has("--seed")) {
        const int64_t seed = a.get_i("--seed", 0);
        used["seed"] = seed;
        if (used.contains("workload")) used["workload"]["seed"] = seed;
    }
    if (a.flag("--no-nvlink")) used["cluster"]["nvlink_available"] = false;
    const std::string dir = a.has("--out") ? a.get("--out") : join_path(output_root(), "run_out");
    json run_cfg = used;
    resolve_trace(run_cfg, config_path);
    const prefixsim::ExperimentConfig cfg = prefixsim::experiment_from_json(run_cfg);  // validates

    if (a.has("--dump-tree")) {
        // index view of the workload: every request pooled at its prompt length
        prefixsim::QuadTree tree;
        const auto reqs = cfg.workload.kind == prefixsim::WorkloadSpec::Kind::kTrace
                              ? prefixsim::ingest_trace(cfg.workload.trace_path, cfg.workload.trace_format).requests
                              : prefixsim::generate_synthetic(cfg.workload);
        for (const auto& r : reqs) {
            tree.insert({r.id, r.prompt_len, prefixsim::blocks_for(r.prompt_len, cfg.sim.cluster.block_size)}, 0.0);
        }
        prefixsim::write_file(a.get("--dump-tree"), tree.dump_json().dump(2) + "\n");
    }

    asv_engine_opts o{};
    o.decode_device = static_cast<int32_t>(a.get_i("--device", 0));
    o.prefetch_device = static_cast<int32_t>(a.get_i("--prefetch-device", o.decode_device));
    shape_of(run_cfg, a, o);
    o.execute_transfers = a.flag("--resident") ? 0 : 1;
    o.execute_prefill_offload = a.flag("--prefill-offload") || o.prefetch_device != o.decode_device ? 1 : 0;
    o.host_pool_bytes = a.get_i("--host-pool-mib", 4096) << 20;
    o.exec_begin = a.get_i("--exec-begin", 0);
    o.exec_end = a.get_i("--exec-end", -1);
    o.timed_begin = a.get_i("--timed-begin", o.exec_begin);
    o.copy_begin = a.get_i("--copy-begin", o.exec_begin);
    o.shard_index = static_cast<int32_t>(a.get_i("--shard", 0));
    o.shard_count = static_cast<int32_t>(a.get_i("--shards", 1));
    o.pdl = 1;
    o.run_ahead = static_cast<int32_t>(a.get_i("--run-ahead", 256));
    o.pair_mode = a.flag("--pair-mode") ? 1 : 0;
    o.full_step = a.flag("--full-step") ? 1 : 0;
    o.intermediate_size = 0;

    asv_engine_stats st{};
    const std::string text = run_cfg.dump();
    if (asv_engine_run_ex(text.c_str(), nullptr, &o, &st, dir.c_str(), nullptr, nullptr) != ASV_OK) {
        throw std::runtime_error(asv_last_error());
    }
    prefixsim::write_file(join_path(dir, "config_used.json"), used.dump(2) + "\n");
    const json summary = json::parse(prefixsim::read_file(join_path(dir, "summary.json")));
    const double measured = st.window_ms > 0 ? static_cast<double>(st.tokens_timed) / (st.window_ms * 1e-3) : 0.0;
    std::cout << "policy " << used.value("policy", std::string("aligned")) << ": "
              << summary.value("completed_requests", int64_t(0)) << " completed, "
              << summary.value("rejected_requests", int64_t(0)) << " rejected, decode throughput "
              << summary.value("decode_throughput_tok_s", 0.0) << " tok/s, TPOT p99 "
              << summary.value("tpot_p99_ms", 0.0) << " ms\n";
    std::cout << "B200: " << st.iterations_timed << " iterations executed, decode " << measured << " tok/s measured, ";
    if (o.full_step) {  // the whole decoder layer stack: weights + KV streamed per window time
        std::cout << "decoder step HBM "
                  << (st.window_ms > 0 ? static_cast<double>(st.attn_bytes + st.weight_bytes) / (st.window_ms * 1e-3) / 1e9
                                       : 0.0);
    } else {
        std::cout << "attention "
                  << (st.attn_ms > 0 ? static_cast<double>(st.attn_bytes) / (st.attn_ms * 1e-3) / 1e9 : 0.0);
    }
    std::cout << " GB/s, KV moved h2d " << st.h2d_bytes << " B, d2h " << st.d2h_bytes + st.offload_bytes << " B, p2p "
              << st.p2p_bytes << " B\n";
    std::cout << "artifacts in " << dir << "\n";
    return 0;
}

int cmd_compare(const Args& a) {
    const std::string config_path = a.get("--config");
    if (config_path.empty()) throw std::invalid_argument("compare: --config is required");
    json j = json::parse(prefixsim::read_file(config_path));
    resolve_trace(j, config_path);
    const prefixsim::ExperimentConfig cfg = prefixsim::experiment_from_json(j);
    std::vector<prefixsim::Policy> policies;
    {
        std::stringstream ss(a.get("--policies", "aligned,fcfs,disagg-fcfs"));
        std::string tok;
        while (std::getline(ss, tok, ',')) policies.push_back(prefixsim::policy_from_string(tok));
    }
    const int seeds = static_cast<int>(a.get_i("--seeds", 5));
    const auto rows = prefixsim::compare_policies(cfg, policies, seeds);
    const std::string dir = a.has("--out") ? a.get("--out") : join_path(output_root(), "compare_out");
    std::ostringstream csv;
    csv << "policy,throughput_mean,throughput_min,throughput_max,tpot_p99_mean,bubble_total_mean,sched_p95_mean\n";
    for (const auto& r : rows) {
        csv << prefixsim::to_string(r.policy) << "," << r.throughput.mean << "," << r.throughput.min << ","
            << r.throughput.max << "," << r.tpot_p99.mean << "," << r.total_bubble.mean << "," << r.sched_p95.mean
            << "\n";
        std::cout << prefixsim::to_string(r.policy) << ": throughput " << r.throughput.mean << " tok/s (min "
                  << r.throughput.min << ", max " << r.throughput.max << "), TPOT p99 " << r.tpot_p99.mean
                  << " ms, bubble " << r.total_bubble.mean << " ms, sched p95 " << r.sched_p95.mean << " ms\n";
    }
    json ratios = json::object();
    for (const auto& r : rows) {
        if (r.policy == prefixsim::Policy::kAligned) continue;
        for (const auto& al : rows) {
            if (al.policy != prefixsim::Policy::kAligned) continue;
            ratios[std::string("aligned_over_") + prefixsim::to_string(r.policy)] = al.throughput.mean / r.throughput.mean;
        }
    }
    prefixsim::write_file(join_path(dir, "compare.csv"), csv.str());
    prefixsim::write_file(join_path(dir, "ratios.json"), ratios.dump(2) + "\n");
    if (a.flag("--gpu")) {
        // every policy of the base seed executed on the GPU: measured decode tokens/s beside the model's
        json measured = json::object();
        for (const auto p : policies) {
            json pj = j;
            pj["policy"] = prefixsim::to_string(p);
            asv_engine_opts o{};
            o.decode_device = o.prefetch_device = static_cast<int32_t>(a.get_i("--device", 0));
            shape_of(pj, a, o);
            o.execute_transfers = a.flag("--resident") ? 0 : 1;
            o.host_pool_bytes = a.get_i("--host-pool-mib", 4096) << 20;
            o.exec_end = -1;
            o.shard_count = 1;
            o.pdl = 1;
            o.run_ahead = 256;
            asv_engine_stats st{};
            const std::string text = pj.dump();
            if (asv_engine_run_ex(text.c_str(), nullptr, &o, &st, nullptr, nullptr, nullptr) != ASV_OK) {
                throw std::runtime_error(asv_last_error());
            }
            const double tok_s = st.window_ms > 0 ? static_cast<double>(st.tokens_timed) / (st.window_ms * 1e-3) : 0.0;
            measured[prefixsim::to_string(p)] = {{"decode_tokens_per_s_measured", tok_s},
                                                 {"virtual_decode_tok_s", st.virtual_decode_tok_s}};
            std::cout << prefixsim::to_string(p) << " on B200: " << tok_s << " tok/s measured\n";
        }
        prefixsim::write_file(join_path(dir, "gpu_measured.json"), measured.dump(2) + "\n");
    }
    std::cout << "artifacts in " << dir << "\n";
    return 0;
}

int cmd_trace_gen(const Args& a) {
    prefixsim::WorkloadSpec spec;
    if (a.has("--spec")) {
        std::vector<std::string> errors;
        spec = prefixsim::workload_from_json(json::parse(prefixsim::read_file(a.get("--spec"))), errors);
        if (!errors.empty()) {
            for (const auto& e : errors) std::cerr << e << "\n";
            return 2;
        }
    } else {
        spec.count = a.get_i("--count", 1000);
        spec.short_ratio = a.has("--short-ratio") ? std::stod(a.get("--short-ratio")) : 0.95;
        spec.seed = static_cast<uint64_t>(a.get_i("--seed", 1));
    }
    const std::string out = a.get("--out");
    if (out.empty()) throw std::invalid_argument("trace-gen: --out is required");
    const auto reqs = prefixsim::generate_synthetic(spec);
    prefixsim::write_file(out, a.get("--format", "jsonl") == "csv" ? prefixsim::trace_to_csv(reqs)
                                                                   : prefixsim::trace_to_jsonl(reqs));
    std::cout << "wrote " << reqs.size() << " requests to " << out << "\n";
    return 0;
}

int cmd_calibrate(const Args& a) {
    if (!a.has("--anchors")) throw std::invalid_argument("calibrate: --anchors is required");
    const auto anchors = prefixsim::anchors_from_json(json::parse(prefixsim::read_file(a.get("--anchors"))));
    prefixsim::ModelSpec spec;
    if (a.has("--model")) spec = prefixsim::model_spec_from_json(json::parse(prefixsim::read_file(a.get("--model"))));
    const auto fit = prefixsim::calibrate(anchors, spec);
    const auto j = prefixsim::calibration_to_json(fit);
    if (a.has("--out")) prefixsim::write_file(a.get("--out"), j.dump(2) + "\n");
    std::cout << j.dump(2) << "\n";
    std::cout << "mean relative error: " << fit.mean_abs_rel_error << ", max: " << fit.max_abs_rel_error << "\n";
    return 0;
}

void usage() {
    std::cerr << "prefix-aware batching, decode path on B200\n"
                 "usage: prefixsim_gpu <run|compare|trace-gen|calibrate> [options]\n"
                 "  run --config X [--policy P] [--seed N] [--out DIR] [--no-nvlink] [--dump-tree PATH]\n"
                 "      [--device D] [--prefetch-device D] [--resident] [--prefill-offload] [--full-step]\n"
                 "      [--exec-begin I] [--exec-end I] [--timed-begin I] [--copy-begin I] [--shard i --shards n]\n"
                 "      [--heads H --kv-heads K --layers L] [--host-pool-mib M] [--pair-mode]\n"
                 "  compare --config X [--policies a,b] [--seeds N] [--out DIR] [--gpu [--resident]]\n"
                 "  trace-gen --out PATH [--spec S | --count N --short-ratio R --seed N] [--format jsonl|csv]\n"
                 "  calibrate --anchors A [--model M] [--out PATH]\n";
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        usage();
        return 2;
    }
    const std::string cmd = argv[1];
    try {
        if (cmd == "run") {
            return cmd_run(parse(argc, argv, 2, {"--no-nvlink", "--resident", "--prefill-offload", "--full-step",
                                                 "--pair-mode"}));
        }
        if (cmd == "compare") return cmd_compare(parse(argc, argv, 2, {"--gpu", "--resident"}));
        if (cmd == "trace-gen") return cmd_trace_gen(parse(argc, argv, 2, {}));
        if (cmd == "calibrate") return cmd_calibrate(parse(argc, argv, 2, {}));
        if (cmd == "-h" || cmd == "--help") {
            usage();
            return 0;
        }
        usage();
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
