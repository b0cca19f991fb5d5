// GPU executor of the decode-iteration hot path (host C++ runtime).
//
// The data plane of one (prefetch, decode) pair: prefixsim::PairOrchestrator
// (include/prefixsim/cluster_sim.hpp; virtual clock => decisions bit-exact with
// the reference) issues typed orders (KvMove, released, prompt_in_place,
// decode_step) and this executor performs each as real work on the B200:
//   * KV pages live in a device page pool (layout: include/asv.h); a request's
//     KV is a list of pages, allocated at prefetch / growth, freed at release;
//   * batch_prefetch / stray_prefetch (reference cluster_sim.hpp:362-366,
//     581-583) -> H2D copies from the pinned host pool on the transfer stream;
//   * admit / evict (NVLink, :517, :551) -> P2P copies between the prefetch and
//     the decode GPU of a pair, or a zero-copy ownership change on one GPU;
//   * spill / flush (PCIe, :529, :541) -> D2H copies back to the host pool;
//   * prefill_offload (PCIe, :285-299) -> D2H copy of the prefilled KV from the
//     prefill GPU into the request's host-pool pages (prefill compute itself is
//     virtual: the source is a resident prefill-output page ring);
//   * every iteration (:476-496) -> CSR page table in SchedulerState::running
//     order, one plan upload, L decode-attention launches (PDL-chained).
// Bytes moved equal the reference's: a request with s tokens moves
// floor(s/16) whole pages plus a 2-D copy of the s%16 valid rows of its last
// page (s * kv_bytes_per_token in total, cluster_sim.hpp:239-241).
//
// Threads and ordering (copy_runtime.h): the engine thread runs the decisions
// and launches iterations on the compute stream; a CopyWorker thread issues
// every copy-stream operation, so a full copy queue never stalls a launch.
// Streams order each other through sequence flags (stream memory ops):
//   * after executed iteration e the compute stream writes kIter = e + 1;
//   * each KV move writes its lane flag (kBulk / kUrgent / kD2H / kP2P) with
//     the next lane sequence number; the compute stream waits for it when the
//     request is admitted;
//   * a copy writing fresh pages waits only for the iteration that last used
//     them (page hazards, oldest-released pages first); D2H / evict copies of
//     running pages wait for the last launched iteration;
//   * pages read by a copy are quarantined until its lane flag passes.
// The host runs ahead of the GPU by at most `run_ahead` iterations (ring of
// events + a plan arena), issuing future boundaries' KV moves early.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <prefixsim/experiment.hpp>
#include <prefixsim/io.hpp>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <thread>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/asv.h"
#include "asv_internal.h"
#include "copy_runtime.h"
#include "engine_internal.h"

namespace asv {

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define ASV_CUDA(call)                                                                    \
    do {                                                                                  \
        cudaError_t asv_e_ = (call);                                                      \
        if (asv_e_ != cudaSuccess)                                                        \
            throw CudaError(std::string(#call) + ": " + cudaGetErrorString(asv_e_));     \
    } while (0)

namespace {

// Fixed pool of physical KV pages on one device.
// Free pages are handed out oldest-released first, each with its hazard: the
// executed-iteration index of the last decode iteration that may still read or
// append to it (-1: none).  A copy writing a fresh page waits only for that
// iteration, not for the whole GPU queue, so prefetches stream back to back.
class PagePool {
 public:
    // `page_bytes`: one page across all layers; `slice`: one layer of one page
    void init(int device, int64_t pages, int64_t page_bytes, int64_t slice, const SeqFlags* flags) {
        device_ = device;
        flags_ = flags;
        pages_ = pages;
        page_bytes_ = page_bytes;
        slice_ = slice;
        ASV_CUDA(cudaSetDevice(device));
        ASV_CUDA(cudaMalloc(&base_, static_cast<size_t>(pages * page_bytes)));
        ASV_CUDA(cudaMemset(base_, 0, static_cast<size_t>(pages * page_bytes)));
        // page ids beyond the last full layer-major group are never handed out
        const int64_t usable = pool_usable_pages(slice, pages);
        for (int64_t p = 0; p < usable; ++p) free_.push_back({static_cast<int32_t>(p), -1});
    }
    ~PagePool() {
        if (base_ != nullptr) {
            cudaSetDevice(device_);
            cudaFree(base_);
        }
    }
    // `hazard` (optional) accumulates the newest iteration the page may still be used by
    int32_t alloc(int64_t* hazard = nullptr) {
        if (free_.empty()) reclaim(true);
        if (free_.empty()) throw std::runtime_error("KV page pool exhausted on device " + std::to_string(device_));
        const FreePage f = free_.front();
        free_.pop_front();
        if (hazard != nullptr) *hazard = std::max(*hazard, f.hazard);
        return f.page;
    }
    void release(const std::vector<int32_t>& pages, int64_t hazard) {
        for (const int32_t p : pages) free_.push_back({p, hazard});
    }
    // pages become reusable once lane flag `slot` reaches `v` (the copy reading them is done)
    void release_after(int slot, uint32_t v, std::vector<int32_t> pages) {
        quarantine_.push_back({slot, v, std::move(pages)});
    }
    void reclaim(bool block) {
        while (!quarantine_.empty()) {
            auto& q = quarantine_.front();
            if (!flags_->reached(q.slot, q.v)) {
                if (!block) break;
                const auto t0 = std::chrono::steady_clock::now();
                while (!flags_->reached(q.slot, q.v)) {
                    // a failed copy worker never writes the flag, nor does a stalled device: throw, do not hang
                    if (health_) health_(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
                    std::this_thread::sleep_for(std::chrono::microseconds(20));
                }
                wait_ms_ += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
                block = false;  // one blocking wait, then drain whatever else finished
            }
            for (const int32_t p : q.pages) free_.push_back({p, -1});  // the copy waited for its readers
            quarantine_.pop_front();
        }
    }
    char* base() const { return base_; }
    int64_t size() const { return pages_; }
    int device() const { return device_; }
    double wait_ms() const { return wait_ms_; }
    // called while spinning on a flag; throws when the thread that would write it has failed
    void set_health_check(std::function<void(double)> f) { health_ = std::move(f); }

 private:
    std::function<void(double)> health_;  // (seconds this wait has lasted)
    struct FreePage {
        int32_t page;
        int64_t hazard;
    };
    struct Q {
        int slot;
        uint32_t v;
        std::vector<int32_t> pages;
    };
    const SeqFlags* flags_ = nullptr;
    int device_ = 0;
    int64_t pages_ = 0, page_bytes_ = 0, slice_ = 0;
    char* base_ = nullptr;
    std::deque<FreePage> free_;
    std::deque<Q> quarantine_;
    double wait_ms_ = 0.0;
};

struct ReqKV {
    enum Where { kHost, kDecode, kPrefetch };
    Where where = kHost;
    std::vector<int32_t> pages;
    int ready_slot = -1;          // lane flag + value of the copy that filled `pages` (-1: none pending)
    uint32_t ready_v = 0;
    int host_slot = -1;           // lane flag + value of the D2H copy (prefill offload, spill, flush) that
    uint32_t host_v = 0;          // last wrote its host-pool pages (-1: none pending)
    int64_t prefix = 0;
};

// Content mode (asv_engine_opts.content_check, a test mode): every KV row and
// every query is a pure function of (global request id, token position,
// layer, K|V|Q, head), so the output of any executed iteration can be checked
// against an independent CPU restatement (oracle/attn_oracle.c,
// asv_oracle_content_attention) without shadowing the page pools: a page moved
// to the wrong place, reused too early, or copied with the wrong byte count
// changes the attention output.  Values are k/128 (k an int8 from splitmix64),
// queries k/8: exact in bf16, and the 16x query scale makes each softmax peak
// on a few keys so one wrong page moves the output by O(1).
namespace content {
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;
inline uint64_t mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
enum Kind { kK = 0, kV = 1, kQ = 2 };
inline uint64_t key(int64_t req, int64_t pos, int layer, int kind, int head) {
    return ((((static_cast<uint64_t>(req) << 21 | static_cast<uint64_t>(pos)) << 6 | static_cast<uint64_t>(layer))
                 << 2 |
             static_cast<uint64_t>(kind))
            << 8) |
           static_cast<uint64_t>(head);
}
// the 128 bf16 values of one row
inline void row(uint64_t k, bool query, uint16_t* out) {
    const uint64_t seed = mix(k + kGolden);
    const float scale = query ? 1.f / 8.f : 1.f / 128.f;
    for (int w = 0; w < 16; ++w) {
        const uint64_t v = mix(seed + static_cast<uint64_t>(w + 1) * kGolden);
        for (int j = 0; j < 8; ++j) {
            const float f = static_cast<float>(static_cast<int8_t>(v >> (8 * j))) * scale;
            uint32_t u;
            std::memcpy(&u, &f, 4);
            out[w * 8 + j] = static_cast<uint16_t>(u >> 16);  // exact: <= 8 significant bits
        }
    }
}
}  // namespace content

// Per-request host-pool pages of content mode (no aliasing): pinned arena, bump
// allocated; a page gets the prompt rows it covers when it is first handed out,
// later rows arrive through the engine's own D2H write-backs.
class ContentStore {
 public:
    void init(char* arena, int64_t arena_pages, int64_t page_bytes, int32_t layers, int32_t n_kv) {
        arena_ = arena;
        cap_ = arena_pages;
        page_bytes_ = page_bytes;
        layers_ = layers;
        n_kv_ = n_kv;
    }
    char* page(int64_t global_id, std::size_t local, int64_t j, int64_t prompt_len) {
        if (local >= pages_.size()) pages_.resize(local + 1);
        auto& v = pages_[local];
        while (static_cast<int64_t>(v.size()) <= j) {
            if (used_ >= cap_) throw std::runtime_error("content mode: host pool exhausted (raise host_pool_bytes)");
            char* p = arena_ + used_++ * page_bytes_;
            const int64_t t0 = static_cast<int64_t>(v.size()) * 16;
            fill(p, global_id, t0, std::min<int64_t>(t0 + 16, prompt_len));
            v.push_back(p);
        }
        return v[static_cast<std::size_t>(j)];
    }

 private:
    // prompt rows [t0, t1) of the page starting at token t0 (page-major host layout, XOR swizzle)
    void fill(char* p, int64_t id, int64_t t0, int64_t t1) const {
        uint16_t r[128];
        for (int64_t t = t0; t < t1; ++t) {
            const int64_t tr = t - t0;
            for (int l = 0; l < layers_; ++l) {
                for (int kv = 0; kv < 2; ++kv) {
                    for (int h = 0; h < n_kv_; ++h) {
                        content::row(content::key(id, t, l, kv, h), false, r);
                        char* blk = p + ((static_cast<int64_t>(l) * 2 + kv) * n_kv_ + h) * 4096 + tr * 256;
                        for (int c = 0; c < 16; ++c) std::memcpy(blk + ((c ^ (tr & 7)) << 4), r + 8 * c, 16);
                    }
                }
            }
        }
    }
    char* arena_ = nullptr;
    int64_t cap_ = 0, used_ = 0, page_bytes_ = 0;
    int32_t layers_ = 0, n_kv_ = 0;
    std::vector<std::vector<char*>> pages_;
};

class GpuExecutor : public prefixsim::DataPlane {
 public:
    GpuExecutor(const asv_engine_opts& o, const prefixsim::SimConfig& sim, const prefixsim::ModelSpec& spec,
                std::size_t num_requests)
        : o_(o), reqs_(num_requests) {
        shape_ = asv_attn_shape{o.num_q_heads, o.num_kv_heads, 128, 16, o.num_layers};
        page_bytes_ = asv_page_bytes(&shape_);
        if (page_bytes_ <= 0) throw std::invalid_argument(asv_last_error());
        row_bytes_all_ = static_cast<int64_t>(o.num_layers) * 2 * o.num_kv_heads * 256;  // one token, all layers
        if (row_bytes_all_ != spec.kv_bytes_per_token()) {
            throw std::invalid_argument("attention shape does not match model kv_bytes_per_token (" +
                                        std::to_string(row_bytes_all_) + " vs " +
                                        std::to_string(spec.kv_bytes_per_token()) + ")");
        }
        pair_ = o.prefetch_device != o.decode_device || o.pair_mode != 0;
        content_ = o.content_check != 0;
        if (content_ && (!o.execute_transfers || o.exec_begin != 0 || o.exec_end >= 0 || o.copy_begin != 0 ||
                         o.full_step || o.execute_prefill_offload)) {
            throw std::invalid_argument(
                "content_check needs execute_transfers, every iteration and KV move executed (exec_begin = "
                "copy_begin = 0, exec_end = -1), attention-only steps and no prefill offload");
        }
        const bool peer = o.prefetch_device != o.decode_device;
        const int64_t bmax = sim.b_max_blocks(), crb = sim.crb_capacity_blocks();
        dec_pages_ = sim.cluster.decode_hbm_blocks + (pair_ ? 0 : bmax + crb) + 64;
        pre_pages_ = pair_ ? bmax + crb + 64 : 0;
        // memory check before committing
        ASV_CUDA(cudaSetDevice(o.decode_device));
        size_t fr = 0, tot = 0;
        ASV_CUDA(cudaMemGetInfo(&fr, &tot));
        if (static_cast<double>(dec_pages_) * page_bytes_ > 0.92 * static_cast<double>(fr)) {
            throw std::invalid_argument("decode page pool (" + std::to_string(dec_pages_) + " pages x " +
                                        std::to_string(page_bytes_) + " B) does not fit free HBM (" +
                                        std::to_string(fr) + " B)");
        }
        slice_ = 2 * static_cast<int64_t>(o.num_kv_heads) * 4096;
        flags_.init();
        serial_ = serial_mode_requested();
        if (stall_limit_s_ <= 0.0) stall_limit_s_ = serial_ ? 3600.0 : 180.0;
        flags_.set_serial(serial_);
        dec_.set_health_check([this](double waited) { check_workers(waited, "page quarantine"); });
        pre_.set_health_check([this](double waited) { check_workers(waited, "page quarantine"); });
        dec_.init(o.decode_device, dec_pages_, page_bytes_, slice_, &flags_);
        if (content_) ASV_CUDA(cudaMemset(dec_.base(), 0xff, static_cast<size_t>(dec_pages_ * page_bytes_)));
        if (pair_ && peer) {
            ASV_CUDA(cudaSetDevice(o.decode_device));
            int can = 0;
            ASV_CUDA(cudaDeviceCanAccessPeer(&can, o.decode_device, o.prefetch_device));
            if (!can) throw std::invalid_argument("decode and prefetch devices have no peer access");
            cudaError_t e = cudaDeviceEnablePeerAccess(o.prefetch_device, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) ASV_CUDA(e);
            cudaGetLastError();
            ASV_CUDA(cudaSetDevice(o.prefetch_device));
            e = cudaDeviceEnablePeerAccess(o.decode_device, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) ASV_CUDA(e);
            cudaGetLastError();
        }
        if (pair_) {
            pre_.init(o.prefetch_device, pre_pages_, page_bytes_, slice_, &flags_);
            if (content_) ASV_CUDA(cudaMemset(pre_.base(), 0xff, static_cast<size_t>(pre_pages_ * page_bytes_)));
        }
        // streams
        ASV_CUDA(cudaSetDevice(o.decode_device));
        ASV_CUDA(cudaStreamCreateWithFlags(&compute_, cudaStreamNonBlocking));
        ASV_CUDA(cudaStreamCreateWithFlags(&p2p_, cudaStreamNonBlocking));
        ASV_CUDA(cudaSetDevice(xfer_device()));
        ASV_CUDA(cudaStreamCreateWithFlags(&xfer_, cudaStreamNonBlocking));
        ASV_CUDA(cudaStreamCreateWithFlags(&xfer2_, cudaStreamNonBlocking));
        ASV_CUDA(cudaStreamCreateWithFlags(&xfer3_, cudaStreamNonBlocking));
        if (const char* nb = std::getenv("ASV_BULK_STREAMS")) n_bulk_ = std::max(1, std::min(3, std::atoi(nb)));
        ASV_CUDA(cudaStreamCreateWithFlags(&d2h_, cudaStreamNonBlocking));  // other PCIe direction
        ASV_CUDA(cudaStreamCreateWithFlags(&urgent_, cudaStreamNonBlocking));  // strays / swap-ins
        ASV_CUDA(cudaStreamCreateWithFlags(&prefill_, cudaStreamNonBlocking));  // prefill offloads (D2H)
        ASV_CUDA(cudaSetDevice(o.decode_device));
        // host pool
        if (o.execute_transfers) {
            arena_pages_ = std::max<int64_t>(1, o.host_pool_bytes / page_bytes_);
            ASV_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&arena_), static_cast<size_t>(arena_pages_ * page_bytes_),
                                   cudaHostAllocPortable));
            std::memset(arena_, 0, static_cast<size_t>(arena_pages_ * page_bytes_));
            if (content_) content_store_.init(arena_, arena_pages_, page_bytes_, o.num_layers, o.num_kv_heads);
            if (o.execute_prefill_offload) {
                // prefill output ring on the prefill (= prefetch) GPU: <= 512 MiB of pages that the
                // offload copies read in rotation (the prefill compute is not executed)
                const int64_t n = std::max<int64_t>(2, std::min<int64_t>(64, (int64_t(512) << 20) / page_bytes_));
                prefill_out_.init(xfer_device(), n, page_bytes_, slice_, &flags_);
                ASV_CUDA(cudaSetDevice(o.decode_device));
            }
        }
        // attention operands
        ASV_CUDA(cudaSetDevice(o.decode_device));
        int32_t workers = 0;
        if (asv_attn_num_workers(&shape_, o.decode_device, &workers) != ASV_OK) throw CudaError(asv_last_error());
        workers_ = workers;
        max_rows_ = std::min<int64_t>(dec_pages_, content_ ? 1024 : 16384);
        const int64_t qbytes = max_rows_ * o.num_q_heads * 256;
        const int64_t kvbytes = max_rows_ * o.num_kv_heads * 256;
        ASV_CUDA(cudaMalloc(&q_, static_cast<size_t>(qbytes)));
        // content mode keeps every layer's output of the iteration (checked against the oracle)
        ASV_CUDA(cudaMalloc(&out_, static_cast<size_t>(qbytes * (content_ ? o.num_layers : 1))));
        if (o.execute_transfers) {  // e2e: every iteration's result lands in host memory
            ASV_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&result_host_), static_cast<size_t>(qbytes),
                                   cudaHostAllocMapped));
        }
        ASV_CUDA(cudaMalloc(&k_new_, static_cast<size_t>(kvbytes)));
        ASV_CUDA(cudaMalloc(&v_new_, static_cast<size_t>(kvbytes)));
        fill_random(q_, qbytes / 2, 11);
        fill_random(k_new_, kvbytes / 2, 12);
        fill_random(v_new_, kvbytes / 2, 13);
        if (o.full_step) init_full_step();
        // Run-ahead ring of in-flight iterations (events, timestamps) and a plan
        // arena: each iteration's plan occupies exactly its size in a circular
        // mapped-host + device arena, so the host can run hundreds of iterations
        // ahead of the GPU (issuing the KV moves of future boundaries early)
        // with bounded memory.  Worst-case plan: every split holds >= 2 pages or
        // is a whole request.
        ring_ = std::max(2, o.run_ahead);
        plan_cap_ = 40 * (dec_pages_ / 2 + max_rows_ + 1) + 2 * max_rows_ + 8;
        plan_scratch_.resize(static_cast<size_t>(plan_cap_ + 4));
        arena_words_ = std::max<int64_t>(2 * (plan_cap_ + 4), int64_t(16) << 20);  // >= 64 MiB
        ASV_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&plan_arena_host_), static_cast<size_t>(arena_words_) * 4,
                               cudaHostAllocMapped));  // pulled by SM loads (asv_plan_upload)
        ASV_CUDA(cudaMalloc(&plan_arena_dev_, static_cast<size_t>(arena_words_) * 4));
        att_beg_.resize(static_cast<size_t>(ring_));
        att_end_.resize(static_cast<size_t>(ring_));
        slot_timed_.assign(static_cast<size_t>(ring_), 0);
        slot_seq_.assign(static_cast<size_t>(ring_), 0);
        slot_b_.assign(static_cast<size_t>(ring_), 0);
        slot_waits_.assign(static_cast<size_t>(ring_), 0);
        if (o.probe_bubble) {
            // per-warp %globaltimer (start, end) of every attention launch of a timed iteration, in
            // device memory; after the iteration one small kernel reduces each launch to (first start,
            // last end, summed busy) in mapped host memory, read at retire
            ASV_CUDA(cudaMalloc(&ts_dev_, static_cast<size_t>(o.num_layers) * workers_ * 16));
            ASV_CUDA(cudaMemset(ts_dev_, 0, static_cast<size_t>(o.num_layers) * workers_ * 16));
            ASV_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&span_host_),
                                   static_cast<size_t>(ring_) * o.num_layers * 3 * 8, cudaHostAllocMapped));
        }
        if (content_) {
            cap_words_ = max_rows_ * o.num_q_heads * 64 * o.num_layers;  // int32 words of one iteration's out
            ASV_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&cap_host_),
                                   static_cast<size_t>(ring_) * static_cast<size_t>(cap_words_) * 4,
                                   cudaHostAllocMapped));
        }
        if (content_ || o.capture_path != nullptr) {
            slot_ids_.assign(static_cast<size_t>(ring_), {});
            slot_lens_.assign(static_cast<size_t>(ring_), {});
        }
        if (o.capture_path != nullptr) {  // content mode: outputs too; otherwise each page table's lengths
            capture_ = std::fopen(o.capture_path, "wb");
            if (capture_ == nullptr) throw std::runtime_error(std::string("cannot open ") + o.capture_path);
        }
        for (int i = 0; i < ring_; ++i) {
            ASV_CUDA(cudaEventCreate(&att_beg_[static_cast<size_t>(i)]));
            ASV_CUDA(cudaEventCreate(&att_end_[static_cast<size_t>(i)]));
        }
        ws_splits_ = static_cast<int32_t>(dec_pages_ / 2 + max_rows_ + 1);
        ws_bytes_ = asv_attn_workspace_bytes(&shape_, 0, ws_splits_);
        ASV_CUDA(cudaMalloc(&ws_, ws_bytes_));
        if (asv_attn_workspace_init(ws_, ws_bytes_, compute_) != ASV_OK) throw CudaError(asv_last_error());
        ASV_CUDA(cudaEventCreate(&win_beg_));
        ASV_CUDA(cudaEventCreate(&win_end_));
        ASV_CUDA(cudaStreamSynchronize(compute_));
        std::memset(stats_.logical_bytes, 0, sizeof(stats_.logical_bytes));
        std::memset(stats_.logical_count, 0, sizeof(stats_.logical_count));
        if (o.execute_transfers) warm_up_copies();
        nvtxInitialize(nullptr);  // NVTX's lazy init is not thread-safe: do it before the workers start
        worker_.start(serial_);
        launcher_.start(serial_);
        if (std::getenv("ASV_WATCHDOG") != nullptr) {
            watchdog_ = std::thread([this] {
                while (!watchdog_stop_.load()) {
                    std::this_thread::sleep_for(std::chrono::seconds(5));
                    std::fprintf(stderr,
                                 "[asv watchdog] executed=%lld phase=%d worker done=%llu queued=%zu in=%s launcher queued=%zu | flags iter=%u "
                                 "bulk=%u/%u urgent=%u/%u d2h=%u/%u p2p=%u/%u\n",
                                 static_cast<long long>(executed_), phase_.load(),
                                 static_cast<unsigned long long>(worker_.done()), worker_.queued(), worker_.current(), launcher_.queued(),
                                 flags_.value(kIter),
                                 flags_.value(kBulk), lane_seq_[kBulk], flags_.value(kUrgent), lane_seq_[kUrgent],
                                 flags_.value(kD2H), lane_seq_[kD2H], flags_.value(kP2P), lane_seq_[kP2P]);
                }
            });
        }
    }

    ~GpuExecutor() override {
        watchdog_stop_.store(true);
        if (watchdog_.joinable()) watchdog_.join();
        // error paths: drop queued copies and release every stream wait on a
        // lane flag that will now never be written, so the device can drain
        launcher_.stop(true);
        worker_.stop(true);
        for (int l = kBulk; l < kLanes; ++l) flags_.force(l, lane_seq_[l]);
        flags_.force(kIter, static_cast<uint32_t>(executed_));
        cudaSetDevice(o_.decode_device);
        cudaDeviceSynchronize();
        if (pair_) {
            cudaSetDevice(o_.prefetch_device);
            cudaDeviceSynchronize();
            cudaSetDevice(o_.decode_device);
        }
        if (plan_arena_host_) cudaFreeHost(plan_arena_host_);
        if (plan_arena_dev_) cudaFree(plan_arena_dev_);
        for (auto e : att_beg_) cudaEventDestroy(e);
        for (auto e : att_end_) cudaEventDestroy(e);
        if (ts_dev_) cudaFree(ts_dev_);
        if (span_host_) cudaFreeHost(span_host_);
        if (cap_host_) cudaFreeHost(cap_host_);
        if (capture_) std::fclose(capture_);
        for (auto& pr : copy_timers_) {
            if (pr.a) cudaEventDestroy(pr.a);
            if (pr.b) cudaEventDestroy(pr.b);
        }
        cudaEventDestroy(win_beg_);
        cudaEventDestroy(win_end_);
        cudaFree(q_);
        cudaFree(out_);
        if (result_host_) cudaFreeHost(result_host_);
        if (weights_) cudaFree(weights_);
        if (h_) cudaFree(h_);
        if (x_) cudaFree(x_);
        if (chain_ws_) asv_linear_chain_ws_destroy(chain_ws_);
        if (act_) cudaFree(act_);
        if (ss_a_) cudaFree(ss_a_);
        if (ss_b_) cudaFree(ss_b_);
        cudaFree(k_new_);
        cudaFree(v_new_);
        cudaFree(ws_);
        if (arena_) cudaFreeHost(arena_);
        cudaStreamDestroy(compute_);
        cudaStreamDestroy(p2p_);
        cudaStreamDestroy(xfer_);
        cudaStreamDestroy(xfer2_);
        cudaStreamDestroy(xfer3_);
        cudaStreamDestroy(d2h_);
        cudaStreamDestroy(urgent_);
        cudaStreamDestroy(prefill_);
    }

    // ------------------------------------------------------- data plane (orders of the orchestrator)
    void released(prefixsim::RequestId id) override {
        const auto t0 = clock_now();
        release_pages(kv(id));
        host_ms_ += ms_since(t0);
    }

    // merged-instance FCFS: the prompt is processed in place on the decode GPU
    void prompt_in_place(prefixsim::RequestId id, int64_t blocks) override {
        const auto t0 = clock_now();
        ReqKV& r = kv(id);
        if (r.pages.empty() && content_) {
            // content mode: the prompt's KV (computed in place by the merged instance) is written into
            // its pages from the content store, so later iterations attend over real rows
            begin_xfer_group(kUrgent);
            fetch_from_host(id, &dec_, /*prefill_in_place=*/true);
            end_xfer_group();
        } else if (r.pages.empty()) {
            r.prefix = blocks * 16;  // only the page count matters for the prompt's KV
            for (int64_t i = 0; i < blocks; ++i) r.pages.push_back(dec_.alloc());
            r.where = ReqKV::kDecode;
        }
        host_ms_ += ms_since(t0);
    }

    void kv_move(const prefixsim::KvMove& m) override {
        const auto t0 = clock_now();
        phase_.store(1);
        const int k = static_cast<int>(m.route);  // KvRoute order == ASV_XFER_* order
        stats_.logical_bytes[k] += m.bytes;
        stats_.logical_count[k] += 1;
        if (!copies_active()) {
            // outside the executed span: keep the page bookkeeping, move nothing
            bookkeep_move(m);
            host_ms_ += ms_since(t0);
            return;
        }
        switch (m.route) {
            case prefixsim::KvRoute::kBatchPrefetch:
                begin_xfer_group();
                for (const auto id : *m.members) fetch_from_host(id, staging_pool());
                end_xfer_group();
                break;
            case prefixsim::KvRoute::kStrayPrefetch:
                begin_xfer_group(kUrgent);
                fetch_from_host(m.request, staging_pool());
                end_xfer_group();
                break;
            case prefixsim::KvRoute::kAdmit:
                if (!aligned_) {
                    // FCFS swap-in / disaggregated admit: host pool -> decode pages (PCIe)
                    begin_xfer_group(kUrgent);
                    fetch_from_host(m.request, &dec_);
                    end_xfer_group();
                } else {
                    admit_to_decode(m.request);  // candidate buffer -> running (NVLink / in place)
                }
                break;
            case prefixsim::KvRoute::kEvict:
                if (!aligned_) {
                    begin_xfer_group(kD2H);
                    write_back_to_host(m.request);
                    end_xfer_group();
                } else {
                    evict_to_prefetch(m.request);
                }
                break;
            case prefixsim::KvRoute::kSpill:
            case prefixsim::KvRoute::kFlush:
                begin_xfer_group(kD2H);
                write_back_to_host(m.request);
                end_xfer_group();
                break;
            case prefixsim::KvRoute::kPrefillOffload:
                if (o_.execute_prefill_offload) {
                    begin_xfer_group(kPrefill);
                    offload_to_host(m.request, m.bytes);
                    end_xfer_group();
                }
                break;
        }
        host_ms_ += ms_since(t0);
        host_copy_ms_ += ms_since(t0);
    }

    void decode_step(const prefixsim::IterationRecord& rec, const std::vector<prefixsim::RunningMember>& running) override {
        const auto t0 = clock_now();
        phase_.store(2);
        ++iterations_total_;
        const int64_t seq = rec.seq;
        const bool exec = seq >= o_.exec_begin && (o_.exec_end < 0 || seq < o_.exec_end);
        // page bookkeeping: every member owns blocks_for(prefix + 1) pages (the
        // step appends its token at index prefix)
        for (const auto& m : running) {
            ReqKV& r = kv(m.id);
            r.prefix = m.prefix_len;
            const int64_t need = (m.prefix_len + 1 + 15) / 16;
            while (static_cast<int64_t>(r.pages.size()) < need) r.pages.push_back(dec_.alloc());
            r.where = ReqKV::kDecode;
        }
        stats_.max_batch = std::max<int64_t>(stats_.max_batch, static_cast<int64_t>(running.size()));
        cur_seq_ = seq + 1;  // decisions from here on belong to the next boundary
        if (!exec) {
            host_ms_ += ms_since(t0);
            return;
        }
        const bool timed = seq >= o_.timed_begin;
        const int64_t e = executed_++;
        last_exec_ = e;
        const size_t slot = static_cast<size_t>(e % ring_);
        // throttle: the slot's previous iteration must be complete before reuse
        if (e >= ring_) retire_through(e - ring_);
        if (static_cast<int64_t>(running.size()) > max_rows_) throw std::runtime_error("batch exceeds q/out rows");

        // CSR page table in running order (= the reference's prefix_lengths order)
        seq_.clear();
        indptr_.assign(1, 0);
        indices_.clear();
        for (const auto& m : running) {
            const ReqKV& r = kv(m.id);
            seq_.push_back(static_cast<int32_t>(m.prefix_len));
            indices_.insert(indices_.end(), r.pages.begin(), r.pages.end());
            indptr_.push_back(static_cast<int32_t>(indices_.size()));
        }
        asv_attn_plan plan{};
        if (asv_attn_plan_build(&shape_, static_cast<int32_t>(running.size()), seq_.data(), indptr_.data(),
                                indices_.data(), workers_, plan_scratch_.data(), plan_cap_, &plan) != ASV_OK) {
            throw std::runtime_error(asv_last_error());
        }
        if (plan.total_splits > ws_splits_) throw std::runtime_error("attention workspace too small");
        check_workers();
        // admitted requests whose KV is still in flight: the iteration waits for it
        std::vector<std::pair<int, uint32_t>> waits;
        for (const auto& m : running) {
            ReqKV& r = kv(m.id);
            if (r.ready_slot >= 0) {
                if (!flags_.reached(r.ready_slot, r.ready_v)) waits.emplace_back(r.ready_slot, r.ready_v);
                r.ready_slot = -1;
            }
        }
        const int64_t ready_waits = static_cast<int64_t>(waits.size());
        // plan (+ for full steps the token positions = prefix lengths, for RoPE; + in content mode
        // the iteration's queries and appended K/V rows of every layer) in one upload
        const int64_t b_rows = static_cast<int64_t>(running.size());
        const int64_t plan_words = (static_cast<int64_t>(plan.total_int32) + 3) & ~int64_t(3);
        const int64_t pos_words = o_.full_step ? b_rows : 0;
        const int64_t q_words = content_ ? b_rows * o_.num_q_heads * 64 : 0;    // [L][b][n_q][128] bf16
        const int64_t kv_words = content_ ? b_rows * o_.num_kv_heads * 64 : 0;  // [L][b][n_kv][128] (K, V)
        const int64_t payload_words =
            ((pos_words + 3) & ~int64_t(3)) + static_cast<int64_t>(o_.num_layers) * (q_words + 2 * kv_words);
        const int64_t pw = plan_region(e, plan_words + payload_words);
        std::memcpy(plan_arena_host_ + pw, plan_scratch_.data(), static_cast<size_t>(plan.total_int32) * 4);
        for (int64_t i = 0; i < pos_words; ++i) plan_arena_host_[pw + plan_words + i] = seq_[static_cast<size_t>(i)];
        if (content_) write_content_payload(running, plan_arena_host_ + pw + plan_words, q_words, kv_words);
        const bool open_window = timed && !window_open_;
        window_open_ = window_open_ || timed;
        const uint32_t launch0 = launches_;
        launches_ += static_cast<uint32_t>(o_.num_layers);
        const bool probe = timed && ts_dev_ != nullptr;
        const int64_t result_bytes = result_host_ ? b_rows * o_.num_q_heads * 256 : 0;
        if (o_.full_step && b_rows > max_rows_full_)
            throw std::runtime_error("full_step: batch exceeds the activation buffers");
        if (content_ || capture_ != nullptr) {
            // what the kernel attends over: each request's seq_len decoded from the split descriptors
            // of the plan being uploaded (running order = the request index of the descriptor)
            slot_ids_[slot].clear();
            slot_lens_[slot].assign(static_cast<size_t>(b_rows), -1);
            for (const auto& m : running) slot_ids_[slot].push_back(global_id(m.id));
            const int32_t* pd = plan_arena_host_ + pw + plan.off_desc;
            for (int32_t g = 0; g < plan.total_splits; ++g) {
                const int32_t r = pd[static_cast<int64_t>(g) * 40], len = pd[static_cast<int64_t>(g) * 40 + 4];
                if (r >= 0 && r < b_rows) slot_lens_[slot][static_cast<size_t>(r)] = len;
            }
            slot_seq_[slot] = seq;
        }
        // The launch worker enqueues the iteration (so a full compute queue never
        // stalls the decisions that issue future KV moves)
        const int64_t upload_words = plan_words + payload_words;
        launcher_.post([this, e, slot, pw, plan, waits = std::move(waits), open_window, launch0, probe, result_bytes,
                        upload_words, plan_words, pos_words, q_words, kv_words, b_rows] {
            ASV_CUDA(cudaSetDevice(o_.decode_device));
            if (open_window) ASV_CUDA(cudaEventRecord(win_beg_, compute_));
            for (const auto& [lane, v] : waits) flags_.wait(compute_, lane, v);
            if (serial_) {  // profilers cannot replay kernels that touch mapped host memory: copy engine
                ASV_CUDA(cudaMemcpyAsync(plan_arena_dev_ + pw, plan_arena_host_ + pw, static_cast<size_t>(upload_words) * 4,
                                         cudaMemcpyHostToDevice, compute_));
            } else if (asv_plan_upload(plan_arena_host_ + pw, plan_arena_dev_ + pw, upload_words, compute_) != ASV_OK) {
                throw CudaError(asv_last_error());
            }
            ASV_CUDA(cudaEventRecord(att_beg_[slot], compute_));
            asv_attn_plan pl = plan;
            asv_attn_args args{};
            args.q = q_;
            args.kv_pool = dec_.base();
            args.pool_pages = dec_.size();
            args.plan_dev = plan_arena_dev_ + pw;
            args.plan = &pl;
            args.k_new = k_new_;
            args.v_new = v_new_;
            args.out = out_;
            args.lse = nullptr;
            args.workspace = ws_;
            args.workspace_bytes = ws_bytes_;
            args.sm_scale = 0.08838834764831845f;
            const int32_t b = pl.batch;
            const int32_t* positions = plan_arena_dev_ + pw + ((pl.total_int32 + 3) & ~3);
            const int32_t* payload = plan_arena_dev_ + pw + plan_words + ((pos_words + 3) & ~int64_t(3));
            void* prev_layer_out = nullptr;
            for (int l = 0; l < o_.num_layers; ++l) {
                // RMSNorm, QKV + RoPE -> q_, k_new_, v_new_ (in chain mode layer l > 0's QKV ran in the previous chain)
                if (o_.full_step && (!chain_ || l == 0)) layer_front(l, b, positions);
                if (content_) {  // this layer's queries / appended rows from the upload, its own output slice
                    const int32_t* lp = payload + static_cast<int64_t>(l) * (q_words + 2 * kv_words);
                    args.q = lp;
                    args.k_new = lp + q_words;
                    args.v_new = lp + q_words + kv_words;
                    args.out = static_cast<char*>(out_) + static_cast<int64_t>(l) * b_rows * o_.num_q_heads * 256;
                }
                // attention-only steps: layer l's split merge runs inside layer l+1's launch (one grid
                // boundary per layer); the last layer keeps its merge kernel.  The full step's O GEMM
                // needs the merged rows at once, so it merges per layer.
                const bool defer = defer_merge_ && !o_.full_step && pl.n_merge > 0;
                args.defer_merge = defer && l + 1 < o_.num_layers ? 1 : 0;
                args.prev_out = defer && l > 0 ? prev_layer_out : nullptr;
                prev_layer_out = args.out;
                args.layer = l;
                args.launch_index = launch0 + static_cast<uint32_t>(l);
                args.warp_timestamps = probe ? ts_dev_ + static_cast<int64_t>(l) * workers_ * 2 : nullptr;
                // layer 0 of attention-only steps reads the plan the upload kernel just wrote
                args.pdl = (l == 0 && !o_.full_step) ? 0 : o_.pdl;
                if (asv_decode_attention(&shape_, &args, compute_) != ASV_OK) throw CudaError(asv_last_error());
                if (o_.full_step) {  // O + residual, RMSNorm, gate/up SiLU, down + residual (+ next layer's QKV)
                    if (chain_) layer_back_chain(l, b, positions);
                    else layer_back(l, b);
                }
            }
            ASV_CUDA(cudaEventRecord(att_end_[slot], compute_));
            if (probe) {  // per launch: first warp start, last warp end, summed warp busy time
                ASV_CUDA(warp_span_reduce(ts_dev_, workers_, o_.num_layers,
                                          span_host_ + slot * static_cast<size_t>(o_.num_layers) * 3, compute_));
            }
            if (content_) {  // every layer's output of the iteration -> its capture slot
                read_back(static_cast<const int32_t*>(out_), cap_host_ + slot * static_cast<size_t>(cap_words_),
                          b_rows * o_.num_q_heads * 64 * o_.num_layers);
            } else if (result_bytes > 0) {  // the step's result (last layer's output / hidden state) read back
                read_back(static_cast<const int32_t*>(o_.full_step ? h_ : out_),
                          reinterpret_cast<int32_t*>(result_host_), result_bytes / 4);
            }
            flags_.write(compute_, kIter, static_cast<uint32_t>(e + 1));  // executed iterations complete
        }, "iteration");
        slot_timed_[slot] = timed ? 1 : 0;
        if (tracing_) {
            slot_seq_[slot] = seq;
            slot_b_[slot] = static_cast<int64_t>(running.size());
            slot_waits_[slot] = ready_waits;
        }
        if (timed) {
            ++stats_.iterations_timed;
            stats_.tokens_timed += static_cast<int64_t>(running.size());
            stats_.attn_launches += o_.num_layers;
            // attention (+ merge) per layer, the plan upload, and the e2e result read-back
            const bool deferred = defer_merge_ && !o_.full_step && plan.n_merge > 0;
            const int64_t merges = plan.n_merge > 0 ? (deferred ? 1 : o_.num_layers) : 0;
            stats_.kernel_launches_timed += o_.num_layers + merges + 1 + (result_bytes > 0 ? 1 : 0) + (probe ? 1 : 0);
            if (o_.full_step) {  // per layer: 2 RMSNorm + 4 linear launches per 256-row chunk
                const int64_t chunks = (static_cast<int64_t>(running.size()) + 255) / 256;
                // RMSNorm launches: 2 per layer unfused; fused, only layer 0's first one remains
                const int64_t norms = fuse_norm_ ? 1 : 2 * o_.num_layers;
                // chain mode: layer 0's QKV + one persistent GEMM-chain launch per layer and chunk
                stats_.kernel_launches_timed += norms + (chain_ ? chunks * (1 + o_.num_layers)
                                                                : o_.num_layers * 4 * chunks);
                stats_.weight_bytes += o_.num_layers * weights_bytes_per_layer_;
            }
            if (first_timed_start_ < 0) first_timed_start_ = rec.start_ms;
            last_timed_end_ms_ = rec.end_ms;
            stats_.bubble_ms_timed += rec.bubble_ms;
            int64_t kv_tokens = 0;
            for (const auto& m : running) kv_tokens += m.prefix_len;
            const int64_t b = static_cast<int64_t>(running.size());
            stats_.attn_bytes += o_.num_layers * (kv_tokens * 2 * o_.num_kv_heads * 256 + b * o_.num_q_heads * 512 +
                                                  b * 2 * o_.num_kv_heads * 256) +
                                 static_cast<int64_t>(plan.total_int32) * 4;
            last_timed_end_ = true;
            stats_.result_d2h_bytes_window += result_bytes;
        }
        host_ms_ += ms_since(t0);
        if (exec) host_iter_ms_ += ms_since(t0);
    }

    void finish(const prefixsim::MetricsLog& log, asv_engine_stats* out) {
        phase_.store(3);
        if (window_open_) {
            launcher_.post([this] {
                ASV_CUDA(cudaSetDevice(o_.decode_device));
                ASV_CUDA(cudaEventRecord(win_end_, compute_));
            }, "window_end");
        }
        launcher_.drain();
        worker_.drain();
        phase_.store(4);
        check_workers();
        ASV_CUDA(cudaSetDevice(o_.decode_device));
        ASV_CUDA(cudaStreamSynchronize(compute_));
        ASV_CUDA(cudaSetDevice(xfer_device()));
        ASV_CUDA(cudaStreamSynchronize(xfer_));
        ASV_CUDA(cudaStreamSynchronize(xfer2_));
        ASV_CUDA(cudaStreamSynchronize(xfer3_));
        ASV_CUDA(cudaStreamSynchronize(d2h_));
        ASV_CUDA(cudaStreamSynchronize(urgent_));
        ASV_CUDA(cudaStreamSynchronize(prefill_));
        ASV_CUDA(cudaSetDevice(o_.decode_device));
        ASV_CUDA(cudaStreamSynchronize(p2p_));
        retire_through(executed_ - 1);
        if (window_open_) {
            float ms = 0.f;
            ASV_CUDA(cudaEventElapsedTime(&ms, win_beg_, win_end_));
            stats_.window_ms = ms;
        }
        std::vector<std::pair<float, float>> pcie;  // PCIe copy groups relative to the window start
        // a pair's PCIe copies run on the prefetch GPU, whose events cannot be timed against the
        // decode GPU's window events: their union is taken relative to the first timed PCIe group
        const bool cross = xfer_device() != o_.decode_device;
        cudaEvent_t anchor = win_beg_;
        if (cross) {
            anchor = nullptr;
            for (const auto& pr : copy_timers_) {
                if (!pr.p2p) {
                    anchor = pr.a;
                    break;
                }
            }
        }
        const float clip = cross ? 1e30f : static_cast<float>(stats_.window_ms);
        for (auto& pr : copy_timers_) {
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, pr.a, pr.b) == cudaSuccess) {
                (pr.p2p ? stats_.p2p_busy_ms : stats_.h2d_busy_ms) += ms;
            }
            float a = 0.f, b = 0.f;
            if (!pr.p2p && window_open_ && anchor != nullptr && cudaEventElapsedTime(&a, anchor, pr.a) == cudaSuccess &&
                cudaEventElapsedTime(&b, anchor, pr.b) == cudaSuccess) {
                pcie.emplace_back(std::max(0.f, a), std::min(b, clip));
                if (tracing_) {
                    trace_.push_back(std::string("{\"copy\":\"") + pr.lane + "\",\"seq\":" + std::to_string(pr.seq) +
                                     ",\"bytes\":" + std::to_string(pr.bytes) + ",\"t0\":" + std::to_string(a) +
                                     ",\"t1\":" + std::to_string(b) + "}");
                }
            }
        }
        cudaGetLastError();
        std::sort(pcie.begin(), pcie.end());
        float cur_a = -1.f, cur_b = -1.f;
        for (const auto& [a, b] : pcie) {
            if (b <= a) continue;
            if (a > cur_b) {
                if (cur_b > cur_a) stats_.pcie_union_ms += cur_b - cur_a;
                cur_a = a;
                cur_b = b;
            } else {
                cur_b = std::max(cur_b, b);
            }
        }
        if (cur_b > cur_a) stats_.pcie_union_ms += cur_b - cur_a;
        stats_.host_wait_ms = host_wait_ms_ + dec_.wait_ms() + (pair_ ? pre_.wait_ms() : 0.0);
        if (tracing_) {
            trace_.push_back("{\"host_wait\":{\"retire\":" + std::to_string(host_wait_ms_) + ",\"plan_arena\":" +
                             std::to_string(arena_wait_ms_) + ",\"reclaim\":" +
                             std::to_string(dec_.wait_ms() + (pair_ ? pre_.wait_ms() : 0.0)) +
                             "},\"host_copy_ms\":" +
                             std::to_string(host_copy_ms_) + ",\"host_iter_ms\":" + std::to_string(host_iter_ms_) +
                             ",\"executed\":" + std::to_string(executed_) + "}");
            if (FILE* f = std::fopen(std::getenv("ASV_TRACE"), "w")) {
                for (const auto& line : trace_) std::fprintf(f, "%s\n", line.c_str());
                std::fclose(f);
            }
        }
        stats_.iterations_total = iterations_total_;
        stats_.measured_idle_frac = span_ns_ > 0 ? 1.0 - busy_ns_ / span_ns_ : 0.0;
        if (!bubble_iters_.empty()) {
            if (o_.bubble_out != nullptr) {
                const int64_t n = std::min<int64_t>(o_.bubble_out_cap, static_cast<int64_t>(bubble_iters_.size()));
                std::copy(bubble_iters_.begin(), bubble_iters_.begin() + n, o_.bubble_out);
            }
            std::vector<double> v = bubble_iters_;
            std::sort(v.begin(), v.end());
            const auto rank = [&v](double p) {  // nearest rank (reference metrics.hpp nearest_rank)
                const auto k = static_cast<std::size_t>(std::ceil(p * static_cast<double>(v.size())));
                return v[std::min(v.size() - 1, k == 0 ? 0 : k - 1)];
            };
            stats_.bubble_p50_ms = rank(0.50);
            stats_.bubble_p90_ms = rank(0.90);
            stats_.bubble_p99_ms = rank(0.99);
            stats_.bubble_max_ms = v.back();
            stats_.bubble_iterations = static_cast<int64_t>(v.size());
        }
        if (capture_ != nullptr) std::fflush(capture_);
        stats_.virtual_window_ms = first_timed_start_ >= 0 ? last_timed_end_ms_ - first_timed_start_ : 0.0;
        stats_.virtual_decode_tok_s = log.iterations.empty() ? 0.0 : prefixsim::decode_throughput(log);
        stats_.host_decide_ms = host_ms_;
        stats_.pages_decode = dec_pages_;
        stats_.pages_prefetch = pre_pages_;
        *out = stats_;
    }

    double& host_ms() { return host_ms_; }

 private:
    using Clock = std::chrono::steady_clock;
    static Clock::time_point clock_now() { return Clock::now(); }
    static double ms_since(Clock::time_point t0) {
        return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
    }

    ReqKV& kv(prefixsim::RequestId id) { return reqs_.at(static_cast<std::size_t>(id)); }
    int xfer_device() const { return pair_ ? o_.prefetch_device : o_.decode_device; }
    PagePool* staging_pool() { return pair_ ? &pre_ : &dec_; }
    bool in_window() const { return window_open_; }
    bool copies_active() const {
        const int64_t begin = std::min(o_.copy_begin, o_.exec_begin);
        return o_.execute_transfers && cur_seq_ >= begin && (o_.exec_end < 0 || cur_seq_ < o_.exec_end);
    }

    // page ownership changes of a move whose bytes are not moved
    void bookkeep_move(const prefixsim::KvMove& m) {
        switch (m.route) {
            case prefixsim::KvRoute::kBatchPrefetch:
                for (const auto id : *m.members) fetch_from_host(id, staging_pool());
                break;
            case prefixsim::KvRoute::kStrayPrefetch: fetch_from_host(m.request, staging_pool()); break;
            case prefixsim::KvRoute::kAdmit:
                if (!aligned_) fetch_from_host(m.request, &dec_);
                else admit_to_decode(m.request);
                break;
            case prefixsim::KvRoute::kEvict:
                if (!aligned_) write_back_to_host(m.request);
                else evict_to_prefetch(m.request);
                break;
            case prefixsim::KvRoute::kSpill:
            case prefixsim::KvRoute::kFlush: write_back_to_host(m.request); break;
            default: break;
        }
    }

 public:
    bool aligned_ = false;  // aligned policy: admits/evicts move between candidate buffers and HBM

 private:
    int64_t cur_seq_ = 0;  // seq of the next iteration (decisions before it belong to its boundary)
    void fill_random(void* dst, int64_t elems, uint64_t seed) {
        std::vector<uint16_t> h(static_cast<size_t>(elems));
        uint64_t s = seed;
        for (auto& v : h) {
            s += 0x9e3779b97f4a7c15ULL;
            uint64_t z = s;
            z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
            z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
            z ^= z >> 31;
            const float f = static_cast<float>(static_cast<double>(z >> 11) * 0x1.0p-53 * 2.0 - 1.0);
            uint32_t u;
            std::memcpy(&u, &f, 4);
            v = static_cast<uint16_t>((u + 0x7fffu + ((u >> 16) & 1u)) >> 16);
        }
        ASV_CUDA(cudaMemcpy(dst, h.data(), static_cast<size_t>(elems) * 2, cudaMemcpyHostToDevice));
    }

    // Copies issued by one decision form a group (one timer pair).  Batch
    // prefetches run on xfer_, small urgent H2D moves (strays, swap-ins) on
    // urgent_ so they never queue behind a whole batch, D2H on d2h_ (both PCIe
    // directions at once), admits/evicts of a pair on p2p_.  Every operation on
    // those streams is posted to the copy worker thread.
    // A batch prefetch is spread over n_bulk_ streams (one request each, round
    // robin): concurrent H2D streams keep more PCIe reads in flight.
    enum Lane { kIter = 0, kBulk = 1, kUrgent = 2, kD2H = 3, kP2P = 4, kBulk2 = 5, kBulk3 = 6, kPrefill = 7,
                kLanes = 8 };
    static_assert(kLanes <= SeqFlags::kSlots, "one sequence flag per lane");
    cudaStream_t lane_stream(int lane) const {
        switch (lane) {
            case kPrefill: return prefill_;
            case kD2H: return d2h_;
            case kUrgent: return urgent_;
            case kP2P: return p2p_;
            case kBulk2: return xfer2_;
            case kBulk3: return xfer3_;
            default: return xfer_;
        }
    }
    int bulk_lane(int64_t i) const {
        static constexpr int kBulkLanes[3] = {kBulk, kBulk2, kBulk3};
        return kBulkLanes[i % n_bulk_];
    }
    int lane_device(int lane) const { return lane == kP2P ? o_.decode_device : xfer_device(); }

    // the lane's stream waits for executed iteration `hz` (skipped when it is
    // known complete, or already awaited on that stream)
    void lane_wait_iteration(int lane, int64_t hz) {
        if (hz < 0 || hz + 1 <= waited_iter_[lane]) return;
        if (flags_.reached(kIter, static_cast<uint32_t>(hz + 1))) return;
        waited_iter_[lane] = hz + 1;
        ++stats_.hazard_waits;
        const cudaStream_t st = lane_stream(lane);
        const int dev = lane_device(lane);
        const uint32_t v = static_cast<uint32_t>(hz + 1);
        worker_.post([this, st, dev, v] {
            ASV_CUDA(cudaSetDevice(dev));
            flags_.wait(st, kIter, v);
        }, "wait_iter");
    }
    // the lane's stream waits for another lane's copy (a request's readiness)
    void lane_wait_ready(int lane, ReqKV& r) {
        if (r.ready_slot < 0) return;
        const int slot = r.ready_slot;
        const uint32_t v = r.ready_v;
        r.ready_slot = -1;
        if (slot == lane || flags_.reached(slot, v)) return;  // same stream: ordered already
        const cudaStream_t st = lane_stream(lane);
        const int dev = lane_device(lane);
        worker_.post([this, st, dev, slot, v] {
            ASV_CUDA(cudaSetDevice(dev));
            flags_.wait(st, slot, v);
        }, "wait_ready");
    }
    // the lane's stream announces everything posted so far: returns the value
    uint32_t lane_signal(int lane) {
        const uint32_t v = ++lane_seq_[lane];
        const cudaStream_t st = lane_stream(lane);
        const int dev = lane_device(lane);
        worker_.post([this, st, dev, lane, v] {
            ASV_CUDA(cudaSetDevice(dev));
            flags_.write(st, lane, v);
        }, "signal");
        return v;
    }
    // timer of `lane` inside the open group: started at the lane's first copy
    void timer_begin(int lane, bool p2p) {
        CopyTimer t{};
        t.p2p = p2p;
        t.lane = lane == kD2H ? 'd' : lane == kUrgent ? 'u' : lane == kP2P ? 'p' : lane == kPrefill ? 'o' : 'b';
        t.seq = cur_seq_;
        t.bytes = 0;
        open_timer_[lane] = static_cast<int64_t>(copy_timers_.size());
        const cudaStream_t st = lane_stream(lane);
        const int dev = lane_device(lane);
        // events are created here (not on the worker) and recorded there
        ASV_CUDA(cudaSetDevice(dev));
        ASV_CUDA(cudaEventCreate(&t.a));
        ASV_CUDA(cudaEventCreate(&t.b));
        ASV_CUDA(cudaSetDevice(o_.decode_device));
        copy_timers_.push_back(t);
        const cudaEvent_t ev = t.a;
        worker_.post([st, dev, ev] {
            ASV_CUDA(cudaSetDevice(dev));
            ASV_CUDA(cudaEventRecord(ev, st));
        }, "timer_a");
    }
    void timer_add(int lane, int64_t bytes) {
        if (open_timer_[lane] >= 0) copy_timers_[static_cast<size_t>(open_timer_[lane])].bytes += bytes;
    }
    void timer_end(int lane) {
        if (open_timer_[lane] < 0) return;
        CopyTimer& t = copy_timers_[static_cast<size_t>(open_timer_[lane])];
        open_timer_[lane] = -1;
        const cudaStream_t st = lane_stream(lane);
        const int dev = lane_device(lane);
        const cudaEvent_t ev = t.b;
        worker_.post([st, dev, ev] {
            ASV_CUDA(cudaSetDevice(dev));
            ASV_CUDA(cudaEventRecord(ev, st));
        }, "timer_b");
    }

    void begin_xfer_group(int lane = kBulk) {
        group_lane_ = lane_ = lane;
        group_timed_ = copies_active() && in_window();
        if (!copies_active()) return;
        // D2H reads pages the last launched iteration may still use; H2D lanes
        // only wait for the hazards of the pages they allocate (fetch_from_host)
        if (lane == kD2H) lane_wait_iteration(kD2H, executed_ - 1);
    }
    // lane of the next copy of the open group (bulk groups rotate over the bulk streams)
    void next_copy_lane() {
        lane_ = group_lane_ == kBulk ? bulk_lane(bulk_rr_++) : group_lane_;
        if (group_timed_ && open_timer_[lane_] < 0) timer_begin(lane_, false);
    }
    void end_xfer_group() {
        if (!copies_active()) return;
        for (int l = 0; l < kLanes; ++l) timer_end(l);
        lane_ = group_lane_;
        if (!group_quarantine_.empty()) {
            const uint32_t v = lane_signal(lane_);
            for (auto& q : group_quarantine_) q.first->release_after(lane_, v, std::move(q.second));
            group_quarantine_.clear();
        }
    }

    char* host_page(prefixsim::RequestId id, int64_t j) {
        if (content_) {
            return content_store_.page(global_id(id), static_cast<std::size_t>(id), j,
                                       (*requests_)[static_cast<std::size_t>(id)].prompt_len);
        }
        const int64_t a = (id * 7919 + j) % arena_pages_;
        return arena_ + a * page_bytes_;
    }

    // post one request's KV move between host pages and device pages (exact
    // bytes) through the C-ABI copy routines (kv_copy.cpp): whole pages as 2-D
    // copies, the valid rows of a partial last page as one 3-D copy
    int64_t post_copy_kv(const std::vector<int32_t>& pages, const PagePool& pool, prefixsim::RequestId id,
                         int64_t tokens, bool to_device) {
        std::vector<void*> host;
        host.reserve(static_cast<size_t>((tokens + 15) / 16));
        for (int64_t j = 0; j < (tokens + 15) / 16; ++j) host.push_back(host_page(id, j));
        const int64_t expect = tokens * row_bytes_all_;
        const cudaStream_t st = lane_stream(lane_);
        const int dev = lane_device(lane_);
        void* base = pool.base();
        const int64_t pool_pages = pool.size();
        worker_.post([this, pages, host = std::move(host), base, pool_pages, tokens, to_device, st, dev, expect] {
            ASV_CUDA(cudaSetDevice(dev));
            int64_t moved = 0;
            const int rc = to_device ? asv_kv_copy_h2d(&shape_, base, pool_pages, pages.data(), tokens,
                                                       const_cast<const void* const*>(host.data()), st, &moved)
                                     : asv_kv_copy_d2h(&shape_, base, pool_pages, pages.data(), tokens, host.data(), st,
                                                       &moved);
            if (rc != ASV_OK) throw CudaError(asv_last_error());
            if (moved != expect) throw std::logic_error("kv copy moved " + std::to_string(moved) + " bytes, expected " +
                                                        std::to_string(expect));
        }, "copy_host");
        return expect;
    }

    void fetch_from_host(prefixsim::RequestId id, PagePool* pool, bool prefill_in_place = false) {
        ReqKV& r = kv(id);
        const prefixsim::Request& q = (*requests_)[static_cast<std::size_t>(id)];
        r.prefix = q.prefix_len;
        release_pages(r);  // (defensive) a request never holds pages while pooled
        const int64_t n = (q.prefix_len + 15) / 16;
        int64_t hz = -1;
        for (int64_t j = 0; j < n; ++j) r.pages.push_back(pool->alloc(&hz));
        r.where = pool == &dec_ ? ReqKV::kDecode : ReqKV::kPrefetch;
        if (!copies_active()) return;
        next_copy_lane();
        lane_wait_iteration(lane_, hz);
        lane_wait_host(lane_, r);
        const int64_t moved = post_copy_kv(r.pages, *pool, id, q.prefix_len, true);
        if (prefill_in_place) {
            stats_.content_inplace_bytes += moved;  // not a reference transfer
        } else {
            timer_add(lane_, moved);
            stats_.h2d_bytes += moved;
            if (group_timed_) stats_.h2d_bytes_window += moved;
        }
        r.ready_slot = lane_;  // this request is usable as soon as its own pages land
        r.ready_v = lane_signal(lane_);
    }

    // prefill_offload: the prefilled KV (s tokens) leaves the prefill GPU for the
    // request's host-pool pages; reference pool_insert happens at its completion
    // (cluster_sim.hpp:285-299, 379-394), so a later fetch of the request waits
    // for this copy (lane_wait_host)
    void offload_to_host(prefixsim::RequestId id, int64_t bytes) {
        if (bytes % row_bytes_all_ != 0) throw std::logic_error("prefill_offload bytes not a whole number of tokens");
        const int64_t tokens = bytes / row_bytes_all_;
        std::vector<int32_t> src(static_cast<size_t>((tokens + 15) / 16));
        const int64_t ring = pool_usable_pages(slice_, prefill_out_.size());
        for (size_t j = 0; j < src.size(); ++j) src[j] = static_cast<int32_t>(static_cast<int64_t>(j) % ring);
        next_copy_lane();
        const int64_t moved = post_copy_kv(src, prefill_out_, id, tokens, false);
        timer_add(lane_, moved);
        stats_.offload_bytes += moved;
        if (group_timed_) stats_.offload_bytes_window += moved;
        ReqKV& r = kv(id);
        r.host_slot = lane_;
        r.host_v = lane_signal(lane_);
    }
    // the lane's stream waits for the D2H copy that last wrote the request's host pages
    void lane_wait_host(int lane, ReqKV& r) {
        const int slot = r.host_slot;
        const uint32_t v = r.host_v;
        r.host_slot = -1;
        if (slot < 0 || flags_.reached(slot, v)) return;
        const cudaStream_t st = lane_stream(lane);
        const int dev = lane_device(lane);
        worker_.post([this, st, dev, slot, v] {
            ASV_CUDA(cudaSetDevice(dev));
            flags_.wait(st, slot, v);
        }, "wait_host");
    }

    void write_back_to_host(prefixsim::RequestId id) {
        ReqKV& r = kv(id);
        const prefixsim::Request& q = (*requests_)[static_cast<std::size_t>(id)];
        PagePool* pool = r.where == ReqKV::kPrefetch ? &pre_ : &dec_;
        if (copies_active() && !r.pages.empty()) {
            next_copy_lane();
            lane_wait_ready(lane_, r);
            const int64_t moved = post_copy_kv(r.pages, *pool, id, q.prefix_len, false);
            timer_add(lane_, moved);
            stats_.d2h_bytes += moved;
            if (group_timed_) stats_.d2h_bytes_window += moved;
            group_quarantine_.push_back({pool, std::move(r.pages)});
            r.pages.clear();
            r.host_slot = lane_;
            r.host_v = lane_signal(lane_);
        } else {
            pool->release(r.pages, pool == &dec_ ? executed_ - 1 : -1);
            r.pages.clear();
        }
        r.ready_slot = -1;
        r.where = ReqKV::kHost;
    }

    void admit_to_decode(prefixsim::RequestId id) {
        ReqKV& r = kv(id);
        if (!pair_ || r.where == ReqKV::kDecode) {
            r.where = ReqKV::kDecode;  // single GPU: ownership change, zero bytes
            return;
        }
        // pair: prefetch GPU -> decode GPU over NVLink
        std::vector<int32_t> dst;
        int64_t hz = -1;
        for (size_t j = 0; j < r.pages.size(); ++j) dst.push_back(dec_.alloc(&hz));
        if (copies_active()) {
            lane_wait_ready(kP2P, r);
            lane_wait_iteration(kP2P, hz);  // destination pages: only the iteration that last used them
            const bool timed = in_window();
            if (timed) timer_begin(kP2P, true);
            const int64_t moved = post_copy_peer(dst, dec_, r.pages, pre_,
                                                 (*requests_)[static_cast<std::size_t>(id)].prefix_len);
            stats_.p2p_bytes += moved;
            if (timed) {
                stats_.p2p_bytes_window += moved;
                timer_add(kP2P, moved);
                timer_end(kP2P);
            }
            const uint32_t v = lane_signal(kP2P);
            pre_.release_after(kP2P, v, std::move(r.pages));
            r.ready_slot = kP2P;
            r.ready_v = v;
        } else {
            pre_.release(r.pages, -1);
        }
        r.pages = std::move(dst);
        r.where = ReqKV::kDecode;
    }

    void evict_to_prefetch(prefixsim::RequestId id) {
        ReqKV& r = kv(id);
        if (!pair_) return;  // single GPU: the pages stay, ownership moves to the buffer
        std::vector<int32_t> dst;
        for (size_t j = 0; j < r.pages.size(); ++j) dst.push_back(pre_.alloc());
        if (copies_active()) {
            lane_wait_iteration(kP2P, executed_ - 1);  // the request ran in the last launched iteration
            const int64_t moved = post_copy_peer(dst, pre_, r.pages, dec_,
                                                 (*requests_)[static_cast<std::size_t>(id)].prefix_len);
            stats_.p2p_bytes += moved;
            if (in_window()) stats_.p2p_bytes_window += moved;
            const uint32_t v = lane_signal(kP2P);
            dec_.release_after(kP2P, v, std::move(r.pages));
            r.ready_slot = kP2P;
            r.ready_v = v;
        } else {
            dec_.release(r.pages, executed_ - 1);
        }
        r.pages = std::move(dst);
        r.where = ReqKV::kPrefetch;
    }

    int64_t post_copy_peer(const std::vector<int32_t>& dst, const PagePool& dpool, const std::vector<int32_t>& src,
                           const PagePool& spool, int64_t tokens) {
        const int64_t expect = tokens * row_bytes_all_;
        const cudaStream_t st = p2p_;
        const int dev = o_.decode_device;
        void* dbase = dpool.base();
        void* sbase = spool.base();
        const int64_t dn = dpool.size(), sn = spool.size();
        const int ddev = dpool.device(), sdev = spool.device();
        worker_.post([this, dst, src, dbase, sbase, dn, sn, ddev, sdev, tokens, st, dev, expect] {
            ASV_CUDA(cudaSetDevice(dev));
            int64_t moved = 0;
            if (asv_kv_copy_d2d(&shape_, dbase, dn, ddev, dst.data(), sbase, sn, sdev, src.data(), tokens, st,
                                &moved) != ASV_OK) {
                throw CudaError(asv_last_error());
            }
            if (moved != expect) throw std::logic_error("kv peer copy moved a wrong byte count");
        }, "copy_peer");
        return expect;
    }

    void release_pages(ReqKV& r) {
        if (r.pages.empty()) return;
        if (r.where == ReqKV::kPrefetch) pre_.release(r.pages, -1);
        else dec_.release(r.pages, executed_ - 1);  // the last launched iteration may still read them
        r.pages.clear();
        r.ready_slot = -1;
        r.where = ReqKV::kHost;
    }

    // One move of every copy shape the run can issue (whole page: 2-D, partial
    // page: 3-D; H2D, D2H, device-local and peer D2D), before any stream waits
    // on a sequence flag: the runtime loads its internal copy kernels lazily at
    // first use, and that load blocks on device-wide progress (a deadlock once
    // a stream is parked on a flag the blocked thread would write; measured).
    void warm_up_copies() {
        const int32_t a[2] = {0, 1}, b[2] = {2, 3};
        const void* host[2] = {arena_, arena_pages_ > 1 ? arena_ + page_bytes_ : arena_};
        int64_t moved = 0;
        ASV_CUDA(cudaSetDevice(xfer_device()));
        PagePool& stage = *staging_pool();
        if (asv_kv_copy_h2d(&shape_, stage.base(), stage.size(), a, 17, host, xfer_, &moved) != ASV_OK ||
            asv_kv_copy_d2h(&shape_, stage.base(), stage.size(), a, 17, const_cast<void* const*>(host), d2h_, &moved) !=
                ASV_OK) {
            throw CudaError(asv_last_error());
        }
        if (o_.execute_prefill_offload &&
            asv_kv_copy_d2h(&shape_, prefill_out_.base(), prefill_out_.size(), a, 17, const_cast<void* const*>(host),
                            prefill_, &moved) != ASV_OK) {
            throw CudaError(asv_last_error());
        }
        ASV_CUDA(cudaStreamSynchronize(xfer_));
        ASV_CUDA(cudaStreamSynchronize(d2h_));
        ASV_CUDA(cudaStreamSynchronize(prefill_));
        ASV_CUDA(cudaSetDevice(o_.decode_device));
        if (asv_kv_copy_d2d(&shape_, dec_.base(), dec_.size(), dec_.device(), b, dec_.base(), dec_.size(),
                            dec_.device(), a, 17, p2p_, &moved) != ASV_OK) {
            throw CudaError(asv_last_error());
        }
        if (pair_ && (asv_kv_copy_d2d(&shape_, dec_.base(), dec_.size(), dec_.device(), a, pre_.base(), pre_.size(),
                                      pre_.device(), a, 17, p2p_, &moved) != ASV_OK ||
                      asv_kv_copy_d2d(&shape_, pre_.base(), pre_.size(), pre_.device(), b, dec_.base(), dec_.size(),
                                      dec_.device(), b, 17, p2p_, &moved) != ASV_OK)) {
            throw CudaError(asv_last_error());
        }
        ASV_CUDA(cudaStreamSynchronize(p2p_));
    }

    // ---------------------------------------------------------------- full decode step
    // Synthetic Llama-style decoder weights (random bf16, fan-in scaled) and the
    // activation buffers of one decode step; the GEMMs run on tcgen05 (asv_linear).
    void init_full_step() {
        hidden_ = o_.num_q_heads * 128;
        inter_ = o_.intermediate_size > 0        ? o_.intermediate_size
                 : hidden_ == 4096 ? 11008 : hidden_ == 5120 ? 13824 : ((hidden_ * 8 / 3 + 127) / 128) * 128;
        if (inter_ % 64 != 0) throw std::invalid_argument("intermediate_size must be a multiple of 64");
        const int64_t n_qkv = 128LL * (o_.num_q_heads + 2 * o_.num_kv_heads);
        const int64_t per_layer = n_qkv * hidden_ + int64_t(hidden_) * hidden_ + 2LL * inter_ * hidden_ +
                                  int64_t(hidden_) * inter_ + 2LL * hidden_;
        max_rows_full_ = std::min<int64_t>(max_rows_, 4096);
        const int64_t rows_pad = (max_rows_full_ + 15) / 16 * 16;
        const int64_t elems = per_layer * o_.num_layers;
        size_t fr = 0, tot = 0;
        ASV_CUDA(cudaMemGetInfo(&fr, &tot));
        const int64_t act = rows_pad * (2LL * hidden_ + inter_) * 2;
        if (static_cast<double>(elems * 2 + act) > 0.9 * static_cast<double>(fr))
            throw std::invalid_argument("full_step: decoder weights do not fit next to the KV pool");
        ASV_CUDA(cudaMalloc(&weights_, static_cast<size_t>(elems) * 2));
        ASV_CUDA(cudaMalloc(&h_, static_cast<size_t>(rows_pad * hidden_ * 2)));
        ASV_CUDA(cudaMalloc(&x_, static_cast<size_t>(rows_pad * hidden_ * 2)));
        ASV_CUDA(cudaMalloc(&act_, static_cast<size_t>(rows_pad * inter_ * 2)));
        ASV_CUDA(cudaMemset(x_, 0, static_cast<size_t>(rows_pad * hidden_ * 2)));
        ASV_CUDA(cudaMemset(act_, 0, static_cast<size_t>(rows_pad * inter_ * 2)));
        weights_bytes_per_layer_ = per_layer * 2;
        auto* w = static_cast<__nv_bfloat16*>(weights_);
        for (int l = 0; l < o_.num_layers; ++l) {
            LayerW lw;
            lw.qkv = w;
            w += n_qkv * hidden_;
            lw.o = w;
            w += int64_t(hidden_) * hidden_;
            lw.gate_up = w;  // tile t: 64 gate rows then the 64 up rows of outputs 64t..64t+63
            w += 2LL * inter_ * hidden_;
            lw.down = w;
            w += int64_t(hidden_) * inter_;
            lw.g1 = w;
            w += hidden_;
            lw.g2 = w;
            w += hidden_;
            const uint64_t sd = 1000 + 16 * static_cast<uint64_t>(l);
            ASV_CUDA(fill_random_bf16(lw.qkv, n_qkv * hidden_, sd, 1.f / std::sqrt(float(hidden_)), 0.f, compute_));
            ASV_CUDA(fill_random_bf16(lw.o, int64_t(hidden_) * hidden_, sd + 1, 1.f / std::sqrt(float(hidden_)), 0.f,
                                      compute_));
            ASV_CUDA(fill_random_bf16(lw.gate_up, 2LL * inter_ * hidden_, sd + 2, 1.f / std::sqrt(float(hidden_)), 0.f,
                                      compute_));
            ASV_CUDA(fill_random_bf16(lw.down, int64_t(hidden_) * inter_, sd + 3, 1.f / std::sqrt(float(inter_)), 0.f,
                                      compute_));
            ASV_CUDA(fill_random_bf16(lw.g1, hidden_, sd + 4, 0.1f, 1.f, compute_));
            ASV_CUDA(fill_random_bf16(lw.g2, hidden_, sd + 5, 0.1f, 1.f, compute_));
            layers_.push_back(lw);
        }
        ASV_CUDA(fill_random_bf16(h_, rows_pad * hidden_, 7, 1.f, 0.f, compute_));
        // fused RMSNorm (asv.h ss_*): the norm weights are folded into the synthetic QKV / gate-up
        // weights and each residual GEMM leaves per-tile row sums of squares for the next GEMM;
        // layer 0 keeps the standalone norm (its input is the step's embedding, not a GEMM output)
        fuse_norm_ = std::getenv("ASV_UNFUSED_NORM") == nullptr;
        ss_parts_ = 2 * (hidden_ / 128);
        ss_ld_ = static_cast<int32_t>(rows_pad);
        ASV_CUDA(cudaMalloc(&ss_a_, static_cast<size_t>(ss_parts_) * rows_pad * 4));
        ASV_CUDA(cudaMalloc(&ss_b_, static_cast<size_t>(ss_parts_) * rows_pad * 4));
        // persistent stream-K chain per layer (decode_chain.cu), opt-in with ASV_LINEAR_CHAIN=1: measured
        // slower than one launch per GEMM (its cross-CTA split-K reduction sits on every phase boundary,
        // DESIGN §4), so the default stays one launch per GEMM with the next weights prefetched into L2
        const char* ce = std::getenv("ASV_LINEAR_CHAIN");
        chain_ = fuse_norm_ && ce != nullptr && std::atoi(ce) != 0;
        if (chain_ && asv_linear_chain_ws_create(o_.decode_device, &chain_ws_) != ASV_OK)
            throw CudaError(asv_last_error());
        ASV_CUDA(cudaStreamSynchronize(compute_));
        if (linear_preload() != cudaSuccess || rmsnorm_preload() != cudaSuccess || linear_chain_preload() != cudaSuccess)
            throw CudaError("full_step: kernel preload failed");
    }

    asv_linear_args lin(const void* w, int32_t n_out, int32_t k, const void* x, int32_t batch, void* y, int32_t y_ld,
                        int32_t epi) const {
        asv_linear_args a{};
        a.w = w;
        a.n_out = n_out;
        a.k = k;
        a.x = x;
        a.x_rows = (batch + 15) / 16 * 16;
        a.batch = batch;
        a.y = y;
        a.y_ld = y_ld;
        a.epilogue = epi;
        a.pdl = o_.pdl;
        return a;
    }
    // GEMMs take <= 256 batch rows per launch
    template <typename F>
    static void row_chunks(int32_t b, F&& f) {
        for (int32_t r0 = 0; r0 < b; r0 += 256) f(r0, std::min<int32_t>(256, b - r0));
    }
    // the weights of the linear launched right after this one (asv.h next_w: with ASV_LINEAR_NEXT_PF the
    // tail of this launch pulls the stages after the next launch's ring into L2)
    static void next_weights(asv_linear_args& a, const void* w, int32_t n_out, int32_t k, int32_t epi) {
        a.next_w = w;
        a.next_n_out = n_out;
        a.next_k = k;
        a.next_epilogue = epi;
    }
    // the next linear takes the raw residual stream h and applies RMSNorm in its epilogue
    void fuse_in(asv_linear_args& a, const float* ss, int32_t r0) const {
        a.ss_in = ss + r0;
        a.ss_parts = ss_parts_;
        a.ss_ld = ss_ld_;
        a.ss_dim = hidden_;
        a.ss_eps = 1e-5f;
    }
    void layer_front(int l, int32_t b, const int32_t* positions) {
        const LayerW& lw = layers_[static_cast<size_t>(l)];
        const int32_t rows = (b + 15) / 16 * 16;
        const bool fused = fuse_norm_ && l > 0;  // ss_a_ holds the previous layer's down-proj sums
        if (!fused && asv_rmsnorm(h_, lw.g1, x_, hidden_, b, rows, 1e-5f, o_.pdl, compute_) != ASV_OK)
            throw CudaError(asv_last_error());
        const auto* xin = static_cast<const __nv_bfloat16*>(fused ? h_ : x_);
        row_chunks(b, [&](int32_t r0, int32_t n) {
            asv_linear_args a = lin(lw.qkv, 128 * (o_.num_q_heads + 2 * o_.num_kv_heads), hidden_,
                                    xin + int64_t(r0) * hidden_, n, nullptr, 0, ASV_EPI_QKV_ROPE);
            if (fused) fuse_in(a, ss_a_, r0);
            a.positions = positions + r0;
            a.rope_theta = 10000.f;
            a.q = static_cast<__nv_bfloat16*>(q_) + int64_t(r0) * o_.num_q_heads * 128;
            a.k_out = static_cast<__nv_bfloat16*>(k_new_) + int64_t(r0) * o_.num_kv_heads * 128;
            a.v_out = static_cast<__nv_bfloat16*>(v_new_) + int64_t(r0) * o_.num_kv_heads * 128;
            a.n_q_heads = o_.num_q_heads;
            a.n_kv_heads = o_.num_kv_heads;
            if (asv_linear(&a, compute_) != ASV_OK) throw CudaError(asv_last_error());
        });
    }
    void layer_back(int l, int32_t b) {
        const LayerW& lw = layers_[static_cast<size_t>(l)];
        const int32_t rows = (b + 15) / 16 * 16;
        auto* h = static_cast<__nv_bfloat16*>(h_);
        row_chunks(b, [&](int32_t r0, int32_t n) {  // h += attn_out . Wo^T
            asv_linear_args a = lin(lw.o, hidden_, hidden_, static_cast<const __nv_bfloat16*>(out_) + int64_t(r0) * hidden_,
                                    n, h + int64_t(r0) * hidden_, hidden_, ASV_EPI_RESIDUAL);
            if (fuse_norm_) {
                a.ss_out = ss_b_ + r0;
                a.ss_ld = ss_ld_;
                next_weights(a, lw.gate_up, 2 * inter_, hidden_, ASV_EPI_SILU_MUL);  // no RMSNorm launch in between
            }
            if (asv_linear(&a, compute_) != ASV_OK) throw CudaError(asv_last_error());
        });
        if (!fuse_norm_ && asv_rmsnorm(h_, lw.g2, x_, hidden_, b, rows, 1e-5f, o_.pdl, compute_) != ASV_OK)
            throw CudaError(asv_last_error());
        auto* act = static_cast<__nv_bfloat16*>(act_);
        const auto* xin = static_cast<const __nv_bfloat16*>(fuse_norm_ ? h_ : x_);
        row_chunks(b, [&](int32_t r0, int32_t n) {  // act = silu(x Wg^T) * (x Wu^T)
            asv_linear_args a = lin(lw.gate_up, 2 * inter_, hidden_, xin + int64_t(r0) * hidden_, n,
                                    act + int64_t(r0) * inter_, inter_, ASV_EPI_SILU_MUL);
            if (fuse_norm_) fuse_in(a, ss_b_, r0);
            next_weights(a, lw.down, hidden_, inter_, ASV_EPI_RESIDUAL);
            if (asv_linear(&a, compute_) != ASV_OK) throw CudaError(asv_last_error());
        });
        row_chunks(b, [&](int32_t r0, int32_t n) {  // h += act . Wd^T
            asv_linear_args a = lin(lw.down, hidden_, inter_, act + int64_t(r0) * inter_, n,
                                    h + int64_t(r0) * hidden_, hidden_, ASV_EPI_RESIDUAL);
            if (fuse_norm_) {  // for the next layer's QKV
                a.ss_out = ss_a_ + r0;
                a.ss_ld = ss_ld_;
                if (l + 1 < o_.num_layers)
                    next_weights(a, layers_[static_cast<size_t>(l + 1)].qkv, 128 * (o_.num_q_heads + 2 * o_.num_kv_heads),
                                 hidden_, ASV_EPI_QKV_ROPE);
            }
            if (asv_linear(&a, compute_) != ASV_OK) throw CudaError(asv_last_error());
        });
    }

    // chain mode: O + residual -> gate/up SiLU -> down + residual -> layer l+1's QKV + RoPE in ONE
    // persistent launch per 256-row chunk (decode_chain.cu); the norms are fused as in layer_back
    void layer_back_chain(int l, int32_t b, const int32_t* positions) {
        const LayerW& lw = layers_[static_cast<size_t>(l)];
        auto* h = static_cast<__nv_bfloat16*>(h_);
        auto* act = static_cast<__nv_bfloat16*>(act_);
        row_chunks(b, [&](int32_t r0, int32_t n) {
            asv_linear_args ph[4];
            ph[0] = lin(lw.o, hidden_, hidden_, static_cast<const __nv_bfloat16*>(out_) + int64_t(r0) * hidden_, n,
                        h + int64_t(r0) * hidden_, hidden_, ASV_EPI_RESIDUAL);
            ph[0].ss_out = ss_b_ + r0;
            ph[0].ss_ld = ss_ld_;
            ph[1] = lin(lw.gate_up, 2 * inter_, hidden_, h + int64_t(r0) * hidden_, n, act + int64_t(r0) * inter_,
                        inter_, ASV_EPI_SILU_MUL);
            fuse_in(ph[1], ss_b_, r0);
            ph[2] = lin(lw.down, hidden_, inter_, act + int64_t(r0) * inter_, n, h + int64_t(r0) * hidden_, hidden_,
                        ASV_EPI_RESIDUAL);
            ph[2].ss_out = ss_a_ + r0;
            ph[2].ss_ld = ss_ld_;
            int nph = 3;
            if (l + 1 < o_.num_layers) {
                const LayerW& nw = layers_[static_cast<size_t>(l + 1)];
                ph[3] = lin(nw.qkv, 128 * (o_.num_q_heads + 2 * o_.num_kv_heads), hidden_, h + int64_t(r0) * hidden_, n,
                            nullptr, 0, ASV_EPI_QKV_ROPE);
                fuse_in(ph[3], ss_a_, r0);
                ph[3].positions = positions + r0;
                ph[3].rope_theta = 10000.f;
                ph[3].q = static_cast<__nv_bfloat16*>(q_) + int64_t(r0) * o_.num_q_heads * 128;
                ph[3].k_out = static_cast<__nv_bfloat16*>(k_new_) + int64_t(r0) * o_.num_kv_heads * 128;
                ph[3].v_out = static_cast<__nv_bfloat16*>(v_new_) + int64_t(r0) * o_.num_kv_heads * 128;
                ph[3].n_q_heads = o_.num_q_heads;
                ph[3].n_kv_heads = o_.num_kv_heads;
                nph = 4;
            }
            if (asv_linear_chain(ph, nph, chain_ws_, compute_) != ASV_OK) throw CudaError(asv_last_error());
        });
    }

    // wall-clock mode: the measured GPU time of the iteration just enqueued (att_beg .. att_end of its
    // slot: plan upload done -> every layer launch of the step complete); blocks until it is known
    bool measured_step_ms(const prefixsim::IterationRecord& rec, double* ms) override {
        if (!o_.wall_clock || last_exec_ < 0 || last_exec_seq_ == rec.seq) return false;
        const bool exec = rec.seq >= o_.exec_begin && (o_.exec_end < 0 || rec.seq < o_.exec_end);
        if (!exec) return false;
        const auto t0 = clock_now();
        last_exec_seq_ = rec.seq;
        launcher_.drain();
        check_workers();
        const size_t slot = static_cast<size_t>(last_exec_ % ring_);
        ASV_CUDA(cudaEventSynchronize(att_end_[slot]));
        float f = 0.f;
        ASV_CUDA(cudaEventElapsedTime(&f, att_beg_[slot], att_end_[slot]));
        *ms = static_cast<double>(f);
        host_ms_ += ms_since(t0);
        return true;
    }

    // device -> mapped pinned host on the compute stream: an SM copy (never queued behind multi-GB
    // copy-engine traffic), or the copy engine in serial mode (profilers cannot replay a kernel that
    // writes mapped host memory)
    void read_back(const int32_t* src, int32_t* dst, int64_t words) {
        if (serial_) {
            ASV_CUDA(cudaMemcpyAsync(dst, src, static_cast<size_t>(words) * 4, cudaMemcpyDeviceToHost, compute_));
        } else {
            ASV_CUDA(sm_copy(src, dst, words, compute_));
        }
    }

    // every host wait loop calls this: a failed worker, or a wait that made no progress for
    // stall_limit_s_ (a device that never writes the awaited flag), ends the run with an error instead
    // of a hang (the destructor then forces every flag so the device drains)
    void check_workers(double waited_s = 0.0, const char* what = "") {
        if (worker_.failed()) throw CudaError("copy worker: " + worker_.error());
        if (launcher_.failed()) throw CudaError("launch worker: " + launcher_.error());
        if (waited_s > stall_limit_s_)
            throw CudaError(std::string("no progress for ") + std::to_string(static_cast<int>(waited_s)) +
                            " s waiting on " + what + " (flags: iter " + std::to_string(flags_.value(kIter)) +
                            ", executed " + std::to_string(executed_) + "); ASV_STALL_TIMEOUT_S raises the limit");
    }

    // global request id of a shard-local one (request i of the trace -> shard i % count, the orchestrator
    // renumbers its requests 0..n-1: cluster_sim.hpp:137-139)
    int64_t global_id(prefixsim::RequestId local) const {
        return static_cast<int64_t>(local) * std::max(1, o_.shard_count) + o_.shard_index;
    }
    // content mode: the iteration's queries and appended K/V rows, [L]{q[b][n_q], k[b][n_kv], v[b][n_kv]}
    void write_content_payload(const std::vector<prefixsim::RunningMember>& running, int32_t* dst, int64_t q_words,
                               int64_t kv_words) const {
        for (int l = 0; l < o_.num_layers; ++l) {
            auto* q = reinterpret_cast<uint16_t*>(dst + static_cast<int64_t>(l) * (q_words + 2 * kv_words));
            uint16_t* k = q + 2 * q_words;
            uint16_t* v = k + 2 * kv_words;
            for (std::size_t r = 0; r < running.size(); ++r) {
                const int64_t id = global_id(running[r].id), s = running[r].prefix_len;
                for (int h = 0; h < o_.num_q_heads; ++h)
                    content::row(content::key(id, s, l, content::kQ, h), true, q + (r * o_.num_q_heads + h) * 128);
                for (int h = 0; h < o_.num_kv_heads; ++h) {
                    content::row(content::key(id, s, l, content::kK, h), false, k + (r * o_.num_kv_heads + h) * 128);
                    content::row(content::key(id, s, l, content::kV, h), false, v + (r * o_.num_kv_heads + h) * 128);
                }
            }
        }
    }
    // content mode: one record of the capture file (asv.h asv_engine_opts.capture_path)
    void write_capture(size_t slot) {
        if (capture_ == nullptr) return;
        const auto& ids = slot_ids_[slot];
        const auto& lens = slot_lens_[slot];
        const int64_t b = static_cast<int64_t>(ids.size());
        const int64_t every = std::max<int64_t>(1, o_.capture_every);
        const int64_t seq = slot_seq_[slot];
        const bool full = seq % every == 0;
        const int32_t hdr[4] = {static_cast<int32_t>(b), o_.num_layers, o_.num_q_heads,
                                !content_ ? -2 : full ? -1 : static_cast<int32_t>(seq % o_.num_q_heads)};
        std::fwrite(&seq, 8, 1, capture_);
        std::fwrite(hdr, 4, 4, capture_);
        std::fwrite(ids.data(), 8, static_cast<size_t>(b), capture_);
        std::fwrite(lens.data(), 4, static_cast<size_t>(b), capture_);
        if (!content_) {  // page-table lengths only
            ++stats_.content_iterations_captured;
            return;
        }
        const auto* out = reinterpret_cast<const uint16_t*>(cap_host_ + slot * static_cast<size_t>(cap_words_));
        if (full) {
            std::fwrite(out, 2, static_cast<size_t>(b * o_.num_q_heads * 128 * o_.num_layers), capture_);
        } else {  // one head of every row and layer: [L][b][128]
            const int h = hdr[3];
            for (int64_t lr = 0; lr < b * o_.num_layers; ++lr)
                std::fwrite(out + (lr * o_.num_q_heads + h) * 128, 2, 128, capture_);
        }
        ++stats_.content_iterations_captured;
    }

    // retire every executed iteration up to and including `e`, in order
    void retire_through(int64_t e) {
        for (; retired_upto_ <= e; ++retired_upto_) retire(retired_upto_);
        while (!live_plans_.empty() && live_plans_.front().first < retired_upto_) live_plans_.pop_front();
    }

    // `words` contiguous words of the plan arena for executed iteration `e`
    // (word offset); waits for the oldest in-flight iterations while their plans
    // still occupy the space
    int64_t plan_region(int64_t e, int64_t words) {
        if (words > arena_words_) throw std::runtime_error("plan larger than the plan arena");
        if (arena_head_ % arena_words_ + words > arena_words_) arena_head_ += arena_words_ - arena_head_ % arena_words_;
        const int64_t begin = arena_head_, end = begin + words;
        // a live plan [b, ...) is overwritten once the new region, one lap back, passes b
        if (!live_plans_.empty() && live_plans_.front().second < end - arena_words_) {
            const auto t0 = clock_now();
            while (!live_plans_.empty() && live_plans_.front().second < end - arena_words_) {
                retire_through(live_plans_.front().first);
            }
            arena_wait_ms_ += ms_since(t0);
        }
        live_plans_.emplace_back(e, begin);
        arena_head_ = end;
        return begin % arena_words_;
    }

    void retire(int64_t e) {
        const size_t slot = static_cast<size_t>(e % ring_);
        if (!flags_.reached(kIter, static_cast<uint32_t>(e + 1))) {
            const auto t0 = clock_now();
            while (!flags_.reached(kIter, static_cast<uint32_t>(e + 1))) {
                check_workers(ms_since(t0) * 1e-3, "an iteration");  // parked on a failed copy lane, or stalled
                std::this_thread::sleep_for(std::chrono::microseconds(20));
            }
            host_wait_ms_ += ms_since(t0);
        }
        if (slot_timed_[slot]) {
            float ms = 0.f;
            ASV_CUDA(cudaEventElapsedTime(&ms, att_beg_[slot], att_end_[slot]));
            stats_.attn_ms += ms;
            if (tracing_) {
                float a = 0.f, b = 0.f;
                ASV_CUDA(cudaEventElapsedTime(&a, win_beg_, att_beg_[slot]));
                ASV_CUDA(cudaEventElapsedTime(&b, win_beg_, att_end_[slot]));
                trace_.push_back("{\"it\":" + std::to_string(slot_seq_[slot]) + ",\"b\":" +
                                 std::to_string(slot_b_[slot]) + ",\"waits\":" + std::to_string(slot_waits_[slot]) +
                                 ",\"t0\":" + std::to_string(a) + ",\"t1\":" + std::to_string(b) + "}");
            }
            slot_timed_[slot] = 0;
            if (span_host_ != nullptr) {  // measured bubble: idle warp time inside each launch's span
                const uint64_t* sp = span_host_ + slot * static_cast<size_t>(o_.num_layers) * 3;  // mapped, complete
                double idle_ms = 0.0;
                for (int l = 0; l < o_.num_layers; ++l) {
                    const uint64_t lo = sp[3 * l], hi = sp[3 * l + 1], busy = sp[3 * l + 2];
                    if (hi <= lo) continue;
                    const double span = static_cast<double>(hi - lo) * workers_;
                    busy_ns_ += static_cast<double>(busy);
                    span_ns_ += span;
                    idle_ms += (span - static_cast<double>(busy)) / workers_ * 1e-6;
                }
                bubble_iters_.push_back(idle_ms);
                stats_.measured_bubble_ms += idle_ms;
            }
        }
        if (capture_ != nullptr) write_capture(slot);
        dec_.reclaim(false);
        if (pair_) pre_.reclaim(false);
    }

 public:
    const std::vector<prefixsim::Request>* requests_ = nullptr;

 private:
    struct CopyTimer {
        cudaEvent_t a = nullptr, b = nullptr;
        bool p2p = false;
        char lane = 'b';       // b bulk H2D, u urgent H2D, d D2H, p P2P (trace only)
        int64_t seq = 0;       // boundary that issued it
        int64_t bytes = 0;
    };
    asv_engine_opts o_;
    asv_attn_shape shape_{};
    int64_t page_bytes_ = 0, row_bytes_all_ = 0, slice_ = 0;
    bool pair_ = false;
    int64_t dec_pages_ = 0, pre_pages_ = 0;
    PagePool dec_, pre_, prefill_out_;
    cudaStream_t compute_ = nullptr, p2p_ = nullptr, xfer_ = nullptr, xfer2_ = nullptr, xfer3_ = nullptr,
                 d2h_ = nullptr, urgent_ = nullptr, prefill_ = nullptr;
    int n_bulk_ = 2;                        // bulk H2D streams (ASV_BULK_STREAMS=1..3)
    int64_t bulk_rr_ = 0;
    int group_lane_ = 1;                    // lane the open group was begun on
    int64_t open_timer_[kLanes] = {-1, -1, -1, -1, -1, -1, -1, -1};  // per lane: timer of the open group
    static_assert(kLanes == 8, "open_timer_ initialiser lists one entry per lane");
    SeqFlags flags_;
    bool serial_ = false;                   // profiler-safe ordering (copy_runtime.h serial mode)
    // host wait without progress that ends the run (s): generous under a profiler (kernel replays)
    double stall_limit_s_ = [] {
        const char* e = std::getenv("ASV_STALL_TIMEOUT_S");
        return e != nullptr ? std::atof(e) : 0.0;
    }();
    int64_t last_exec_ = -1;                // executed-iteration index of the latest decode_step
    int64_t last_exec_seq_ = -1;            // wall clock: seq whose measured time was reported
    CopyWorker worker_;                     // issues every copy-stream operation
    CopyWorker launcher_;                   // issues every compute-stream operation (iterations)
    std::thread watchdog_;                  // ASV_WATCHDOG=1: progress report every 5 s (debugging)
    std::atomic<bool> watchdog_stop_{false};
    std::atomic<int> phase_{0};             // 1 decide/copy, 2 iteration launch, 3 finish
    int lane_ = kBulk;                      // lane of the open copy group
    uint32_t lane_seq_[kLanes] = {};         // last value each lane announced
    int64_t waited_iter_[kLanes] = {};       // iteration flag value each lane's stream already waits for
    char* arena_ = nullptr;
    int64_t arena_pages_ = 1;
    int32_t workers_ = 0;
    int64_t max_rows_ = 0;
    char* result_host_ = nullptr;           // mapped pinned: per-iteration result read-back (e2e)
    // full decode step (o_.full_step)
    struct LayerW {
        __nv_bfloat16 *qkv = nullptr, *o = nullptr, *gate_up = nullptr, *down = nullptr, *g1 = nullptr, *g2 = nullptr;
    };
    std::vector<LayerW> layers_;
    void *weights_ = nullptr, *h_ = nullptr, *x_ = nullptr, *act_ = nullptr;
    float *ss_a_ = nullptr, *ss_b_ = nullptr;  // fused RMSNorm: per-tile row sums of squares of h
    int32_t ss_parts_ = 0, ss_ld_ = 0;
    bool fuse_norm_ = false;
    bool chain_ = false;                          // full step: one persistent GEMM chain per layer
    bool defer_merge_ = std::getenv("ASV_DEFER_MERGE") == nullptr || std::atoi(std::getenv("ASV_DEFER_MERGE")) != 0;
    asv_linear_chain_ws* chain_ws_ = nullptr;
    int32_t hidden_ = 0, inter_ = 0;
    int64_t max_rows_full_ = 0, weights_bytes_per_layer_ = 0;
    void *q_ = nullptr, *out_ = nullptr, *k_new_ = nullptr, *v_new_ = nullptr, *ws_ = nullptr;
    size_t ws_bytes_ = 0;
    int32_t ws_splits_ = 0;
    int ring_ = 16;
    int64_t plan_cap_ = 0;
    std::vector<int32_t> plan_scratch_;
    int32_t *plan_arena_host_ = nullptr, *plan_arena_dev_ = nullptr;
    int64_t arena_words_ = 0, arena_head_ = 0;   // absolute word counter (position = head % arena)
    std::deque<std::pair<int64_t, int64_t>> live_plans_;  // (executed index, absolute begin) in issue order
    int64_t retired_upto_ = 0;                   // every executed iteration below this is retired
    uint64_t* ts_dev_ = nullptr;     // probe_bubble: [L][workers][2] per-warp %globaltimer of one iteration
    uint64_t* span_host_ = nullptr;  // probe_bubble: [ring][L][3] (first start, last end, busy sum), mapped
    std::vector<double> bubble_iters_;  // measured bubble (ms) of every timed iteration
    bool content_ = false;           // content_check test mode
    ContentStore content_store_;
    int32_t* cap_host_ = nullptr;    // content: [ring][L][rows][n_q][128] bf16 outputs, mapped
    int64_t cap_words_ = 0;
    FILE* capture_ = nullptr;
    std::vector<std::vector<int64_t>> slot_ids_;
    std::vector<std::vector<int32_t>> slot_lens_;
    std::vector<cudaEvent_t> att_beg_, att_end_;
    std::vector<int> slot_timed_;
    cudaEvent_t win_beg_ = nullptr, win_end_ = nullptr;
    bool window_open_ = false, last_timed_end_ = false, group_timed_ = false;
    std::vector<ReqKV> reqs_;
    std::vector<std::pair<PagePool*, std::vector<int32_t>>> group_quarantine_;
    std::vector<CopyTimer> copy_timers_;  // events created by the engine thread, recorded by the worker
    std::vector<int32_t> seq_, indptr_, indices_;
    int64_t executed_ = 0, iterations_total_ = 0;
    uint32_t launches_ = 0;
    double host_ms_ = 0.0, host_wait_ms_ = 0.0, arena_wait_ms_ = 0.0;
    double host_copy_ms_ = 0.0, host_iter_ms_ = 0.0;  // trace: issue cost of copies / executed iterations
    // ASV_TRACE=<file>: per timed iteration / copy group GPU start-end (ms from the window start)
    const bool tracing_ = std::getenv("ASV_TRACE") != nullptr;
    std::vector<std::string> trace_;
    std::vector<int64_t> slot_seq_, slot_b_, slot_waits_;
    double first_timed_start_ = -1.0, last_timed_end_ms_ = 0.0;

    double busy_ns_ = 0.0, span_ns_ = 0.0;
    asv_engine_stats stats_{};
};

}  // namespace

// `log_out` (optional) receives the run's decision log (the reference's MetricsLog,
// virtual clock): it is byte-identical to the reference's for the same config
int engine_run(const char* config_json, const char* policy_override, const asv_engine_opts* opts,
               asv_engine_stats* stats, prefixsim::MetricsLog* log_out) {
    try {
        if (config_json == nullptr || opts == nullptr || stats == nullptr) {
            return fail(ASV_ERR_INVALID, "null config/opts/stats");
        }
        prefixsim::ExperimentConfig cfg = prefixsim::experiment_from_json(prefixsim::json::parse(config_json));
        if (policy_override != nullptr) cfg.sim.policy = prefixsim::policy_from_string(policy_override);
        const prefixsim::CalibratedCostModel model =
            cfg.has_calibration ? cfg.calibration
                                : prefixsim::calibrate(prefixsim::reference_mixed_batch_anchors(), cfg.model).model;
        std::vector<prefixsim::Request> reqs = load_workload(cfg);
        shard_requests(reqs, opts->shard_index, std::max(1, opts->shard_count));
        if (reqs.empty()) return fail(ASV_ERR_INVALID, "empty shard");
        prefixsim::PairOrchestrator sim(cfg.sim, model, reqs);
        GpuExecutor ex(*opts, cfg.sim, model.spec, reqs.size());
        ex.requests_ = &sim.requests();
        ex.aligned_ = cfg.sim.policy == prefixsim::Policy::kAligned;
        sim.attach(&ex);
        const auto t0 = std::chrono::steady_clock::now();
        prefixsim::MetricsLog log = sim.run();
        (void)t0;
        ex.finish(log, stats);
        if (log_out != nullptr) *log_out = std::move(log);
        return ASV_OK;
    } catch (const CudaError& e) {
        return fail(ASV_ERR_CUDA, e.what());
    } catch (const std::invalid_argument& e) {
        return fail(ASV_ERR_INVALID, e.what());
    } catch (const std::logic_error& e) {
        return fail(ASV_ERR_LOGIC, e.what());
    } catch (const std::exception& e) {
        return fail(ASV_ERR_RUNTIME, e.what());
    }
}

}  // namespace asv

extern "C" int asv_engine_run(const char* config_json, const char* policy_override, const asv_engine_opts* opts,
                              asv_engine_stats* stats) {
    return asv::engine_run(config_json, policy_override, opts, stats, nullptr);
}

namespace {

std::string stats_to_json(const asv_engine_stats& s) {
    static const char* kinds[ASV_XFER_KINDS] = {"prefill_offload", "batch_prefetch", "stray_prefetch", "admit",
                                                "evict", "spill", "flush"};
    prefixsim::json lb, lc;
    for (int k = 0; k < ASV_XFER_KINDS; ++k) {
        lb[kinds[k]] = s.logical_bytes[k];
        lc[kinds[k]] = s.logical_count[k];
    }
    const double tok_s = s.window_ms > 0 ? static_cast<double>(s.tokens_timed) / (s.window_ms * 1e-3) : 0.0;
    prefixsim::json j = {
        {"decode_tokens_per_s_measured", tok_s},
        {"iterations_total", s.iterations_total},
        {"iterations_timed", s.iterations_timed},
        {"tokens_timed", s.tokens_timed},
        {"window_ms", s.window_ms},
        {"attn_ms", s.attn_ms},
        {"attn_bytes", s.attn_bytes},
        {"attn_hbm_gbps", s.weight_bytes == 0 && s.attn_ms > 0
                              ? static_cast<double>(s.attn_bytes) / (s.attn_ms * 1e-3) / 1e9 : 0.0},
        {"weight_bytes", s.weight_bytes},
        {"decoder_step_hbm_gbps", s.weight_bytes > 0 && s.window_ms > 0
                                      ? static_cast<double>(s.attn_bytes + s.weight_bytes) / (s.window_ms * 1e-3) / 1e9
                                      : 0.0},
        {"h2d_bytes", s.h2d_bytes},
        {"d2h_bytes", s.d2h_bytes},
        {"p2p_bytes", s.p2p_bytes},
        {"offload_bytes", s.offload_bytes},
        {"pcie_union_ms", s.pcie_union_ms},
        {"logical_bytes", lb},
        {"logical_count", lc},
        {"virtual_decode_tok_s", s.virtual_decode_tok_s},
        {"max_batch", s.max_batch},
        {"kernel_launches_timed", s.kernel_launches_timed},
        {"measured_idle_frac", s.measured_idle_frac},
        {"host_decide_ms", s.host_decide_ms},
    };
    return j.dump(2) + "\n";
}

}  // namespace

extern "C" int asv_engine_run_ex(const char* config_json, const char* policy_override, const asv_engine_opts* opts,
                                 asv_engine_stats* stats, const char* out_dir, char** log_out, int64_t* log_len) {
    prefixsim::MetricsLog log;
    const int rc = asv::engine_run(config_json, policy_override, opts, stats, &log);
    if (rc != ASV_OK) return rc;
    try {
        std::string jsonl;
        if (log_out != nullptr || out_dir != nullptr) jsonl = prefixsim::log_to_jsonl(log);
        if (out_dir != nullptr) {
            // the reference's run artefacts (prefixsim_main.cpp write_run_artifacts; SVG charts omitted)
            const std::string d(out_dir);
            const prefixsim::Summary sum = prefixsim::summarize(log);
            prefixsim::write_file(d + "/log.jsonl", jsonl);
            prefixsim::write_file(d + "/summary.json", prefixsim::summary_to_json(sum).dump(2) + "\n");
            prefixsim::write_file(d + "/ttft_cdf.csv", prefixsim::cdf_to_csv(sum.ttft_cdf, "ttft_ms"));
            prefixsim::write_file(d + "/sched_cdf.csv", prefixsim::cdf_to_csv(sum.sched_time_cdf, "schedule_ms"));
            prefixsim::write_file(d + "/gpu_stats.json", stats_to_json(*stats));
        }
        if (log_out != nullptr) {
            char* buf = static_cast<char*>(std::malloc(jsonl.size() + 1));
            if (buf == nullptr) throw std::runtime_error("out of host memory");
            std::memcpy(buf, jsonl.data(), jsonl.size());
            buf[jsonl.size()] = 0;
            *log_out = buf;
            if (log_len != nullptr) *log_len = static_cast<int64_t>(jsonl.size());
        }
        return ASV_OK;
    } catch (const std::exception& e) {
        return asv::fail(ASV_ERR_RUNTIME, e.what());
    }
}
