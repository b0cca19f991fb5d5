// ThreadSanitizer driver of the 3-thread host runtime (csrc/executor.cpp + copy_runtime.h): runs
// asv_engine_run on a config with every KV move executed (engine thread: decisions + plans; copy
// worker: every copy-stream operation; launch worker: every iteration), optionally on the pair data
// path, with the host objects built -fsanitize=thread (tools/tsan/Makefile).  Usage:
//   engine_tsan <config.json> <num_layers> [pair_mode] [run_ahead]
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <sstream>
#include <string>

#include "asv.h"

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: %s <config.json> <num_layers> [pair_mode] [run_ahead]\n", argv[0]);
        return 2;
    }
    std::ifstream f(argv[1]);
    std::stringstream ss;
    ss << f.rdbuf();
    const std::string cfg = ss.str();
    asv_engine_opts o{};
    o.decode_device = 0;
    o.prefetch_device = 0;
    o.num_q_heads = 32;
    o.num_kv_heads = 32;
    o.num_layers = std::atoi(argv[2]);
    o.execute_transfers = 1;
    o.host_pool_bytes = 1LL << 30;
    o.exec_begin = 0;
    o.exec_end = -1;
    o.timed_begin = 0;
    o.shard_index = 0;
    o.shard_count = 1;
    o.pdl = 1;
    o.run_ahead = argc > 4 ? std::atoi(argv[4]) : 8;
    o.copy_begin = 0;
    o.pair_mode = argc > 3 ? std::atoi(argv[3]) : 0;
    o.execute_prefill_offload = 1;
    asv_engine_stats st{};
    const int rc = asv_engine_run(cfg.c_str(), nullptr, &o, &st);
    if (rc != ASV_OK) {
        std::fprintf(stderr, "asv_engine_run failed: %s\n", asv_last_error());
        return 1;
    }
    std::printf("ok: %lld iterations, h2d %lld B, d2h %lld B, p2p %lld B, offload %lld B\n",
                static_cast<long long>(st.iterations_total), static_cast<long long>(st.h2d_bytes),
                static_cast<long long>(st.d2h_bytes), static_cast<long long>(st.p2p_bytes),
                static_cast<long long>(st.offload_bytes));
    return 0;
}
