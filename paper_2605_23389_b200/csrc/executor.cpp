// GPU executor of the decode-iteration hot path (host C++ runtime).
//
// Subscribes to the reference-API engine (prefixsim::Simulation, virtual
// clock => decisions bit-exact with the reference) and performs every decision
// as real work on the B200:
//   * KV pages live in a device page pool (layout: include/asv.h); a request's
//     KV is a list of pages, allocated at prefetch / growth, freed at release;
//   * batch_prefetch / stray_prefetch (reference cluster_sim.hpp:362-366,
//     581-583) -> H2D copies from the pinned host pool on the transfer stream;
//   * admit / evict (NVLink, :517, :551) -> P2P copies between the prefetch and
//     the decode GPU of a pair, or a zero-copy ownership change on one GPU;
//   * spill / flush (PCIe, :529, :541) -> D2H copies back to the host pool;
//   * every iteration (:476-496) -> CSR page table in SchedulerState::running
//     order, one plan upload, L decode-attention launches (PDL-chained).
// Bytes moved equal the reference's: a request with s tokens moves
// floor(s/16) whole pages plus a 2-D copy of the s%16 valid rows of its last
// page (s * kv_bytes_per_token in total, cluster_sim.hpp:239-241).
//
// Ordering: the transfer stream waits on the last launched iteration before
// touching pages (reuse after release / reads for spill); the compute stream
// waits on a request's copy event when it is admitted; pages freed by a copy
// are quarantined until that copy's event completes.  The host runs ahead of
// the GPU by at most `run_ahead` iterations (ring of plan buffers and events).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <prefixsim/experiment.hpp>
#include <prefixsim/io.hpp>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <deque>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/asv.h"
#include "asv_internal.h"
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

int xfer_kind(const std::string& k) {
    if (k == "prefill_offload") return ASV_XFER_PREFILL_OFFLOAD;
    if (k == "batch_prefetch") return ASV_XFER_BATCH_PREFETCH;
    if (k == "stray_prefetch") return ASV_XFER_STRAY_PREFETCH;
    if (k == "admit") return ASV_XFER_ADMIT;
    if (k == "evict") return ASV_XFER_EVICT;
    if (k == "spill") return ASV_XFER_SPILL;
    if (k == "flush") return ASV_XFER_FLUSH;
    return -1;
}

// Fixed pool of physical KV pages on one device.
class PagePool {
 public:
    // `page_bytes`: one page across all layers; `slice`: one layer of one page
    void init(int device, int64_t pages, int64_t page_bytes, int64_t slice) {
        device_ = device;
        pages_ = pages;
        page_bytes_ = page_bytes;
        slice_ = slice;
        ASV_CUDA(cudaSetDevice(device));
        ASV_CUDA(cudaMalloc(&base_, static_cast<size_t>(pages * page_bytes)));
        ASV_CUDA(cudaMemset(base_, 0, static_cast<size_t>(pages * page_bytes)));
        free_.reserve(static_cast<size_t>(pages));
        for (int64_t p = pages - 1; p >= 0; --p) free_.push_back(static_cast<int32_t>(p));
    }
    ~PagePool() {
        if (base_ != nullptr) {
            cudaSetDevice(device_);
            cudaFree(base_);
        }
    }
    int32_t alloc() {
        if (free_.empty()) reclaim(true);
        if (free_.empty()) throw std::runtime_error("KV page pool exhausted on device " + std::to_string(device_));
        const int32_t p = free_.back();
        free_.pop_back();
        return p;
    }
    void release(const std::vector<int32_t>& pages) { free_.insert(free_.end(), pages.begin(), pages.end()); }
    // pages become reusable once `ev` (a copy reading them) has completed
    void release_after(cudaEvent_t ev, std::vector<int32_t> pages) { quarantine_.push_back({ev, std::move(pages)}); }
    void reclaim(bool block) {
        while (!quarantine_.empty()) {
            auto& q = quarantine_.front();
            if (block) {
                ASV_CUDA(cudaEventSynchronize(q.ev));
                block = false;  // one blocking wait, then drain whatever else finished
            } else if (cudaEventQuery(q.ev) != cudaSuccess) {
                break;
            }
            free_.insert(free_.end(), q.pages.begin(), q.pages.end());
            quarantine_.pop_front();
        }
    }
    // layer-0 slice of page p (layer l is l * size() * slice bytes further)
    char* page(int32_t p) const { return base_ + static_cast<int64_t>(p) * slice_; }
    char* base() const { return base_; }
    int64_t size() const { return pages_; }
    int device() const { return device_; }

 private:
    struct Q {
        cudaEvent_t ev;
        std::vector<int32_t> pages;
    };
    int device_ = 0;
    int64_t pages_ = 0, page_bytes_ = 0, slice_ = 0;
    char* base_ = nullptr;
    std::vector<int32_t> free_;
    std::deque<Q> quarantine_;
};

// Ring of reusable events recorded on one stream.
class EventRing {
 public:
    void init(int device, int n) {
        ASV_CUDA(cudaSetDevice(device));
        ev_.resize(static_cast<size_t>(n));
        for (auto& e : ev_) ASV_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    ~EventRing() {
        for (auto e : ev_) cudaEventDestroy(e);
    }
    // record on `st`; the slot's previous recording must have completed (it is
    // older than the ring, so in stream order it has)
    cudaEvent_t record(cudaStream_t st) {
        cudaEvent_t e = ev_[next_++ % ev_.size()];
        ASV_CUDA(cudaEventSynchronize(e));
        ASV_CUDA(cudaEventRecord(e, st));
        return e;
    }

 private:
    std::vector<cudaEvent_t> ev_;
    size_t next_ = 0;
};

struct ReqKV {
    enum Where { kHost, kDecode, kPrefetch };
    Where where = kHost;
    std::vector<int32_t> pages;
    cudaEvent_t ready = nullptr;  // copy that filled `pages` (nullptr: nothing pending)
    int64_t prefix = 0;
};

class GpuExecutor : public prefixsim::EngineObserver {
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
        dec_.init(o.decode_device, dec_pages_, page_bytes_, slice_);
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
        if (pair_) pre_.init(o.prefetch_device, pre_pages_, page_bytes_, slice_);
        // streams
        ASV_CUDA(cudaSetDevice(o.decode_device));
        ASV_CUDA(cudaStreamCreateWithFlags(&compute_, cudaStreamNonBlocking));
        ASV_CUDA(cudaStreamCreateWithFlags(&p2p_, cudaStreamNonBlocking));
        ASV_CUDA(cudaSetDevice(xfer_device()));
        ASV_CUDA(cudaStreamCreateWithFlags(&xfer_, cudaStreamNonBlocking));
        ASV_CUDA(cudaStreamCreateWithFlags(&d2h_, cudaStreamNonBlocking));  // other PCIe direction
        ASV_CUDA(cudaStreamCreateWithFlags(&urgent_, cudaStreamNonBlocking));  // strays / swap-ins
        xfer_ev_.init(xfer_device(), 4096);
        d2h_ev_.init(xfer_device(), 4096);
        urgent_ev_.init(xfer_device(), 4096);
        ASV_CUDA(cudaSetDevice(o.decode_device));
        p2p_ev_.init(o.decode_device, 4096);
        // host pool
        if (o.execute_transfers) {
            arena_pages_ = std::max<int64_t>(1, o.host_pool_bytes / page_bytes_);
            ASV_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&arena_), static_cast<size_t>(arena_pages_ * page_bytes_),
                                   cudaHostAllocPortable));
            std::memset(arena_, 0, static_cast<size_t>(arena_pages_ * page_bytes_));
        }
        // attention operands
        ASV_CUDA(cudaSetDevice(o.decode_device));
        int32_t workers = 0;
        if (asv_attn_num_workers(&shape_, o.decode_device, &workers) != ASV_OK) throw CudaError(asv_last_error());
        workers_ = workers;
        max_rows_ = std::min<int64_t>(dec_pages_, 16384);
        const int64_t qbytes = max_rows_ * o.num_q_heads * 256;
        const int64_t kvbytes = max_rows_ * o.num_kv_heads * 256;
        ASV_CUDA(cudaMalloc(&q_, static_cast<size_t>(qbytes)));
        ASV_CUDA(cudaMalloc(&out_, static_cast<size_t>(qbytes)));
        ASV_CUDA(cudaMalloc(&k_new_, static_cast<size_t>(kvbytes)));
        ASV_CUDA(cudaMalloc(&v_new_, static_cast<size_t>(kvbytes)));
        fill_random(q_, qbytes / 2, 11);
        fill_random(k_new_, kvbytes / 2, 12);
        fill_random(v_new_, kvbytes / 2, 13);
        // plan ring: every split holds >= 2 pages or is a whole request
        ring_ = std::max(2, o.run_ahead);
        plan_cap_ = 40 * (dec_pages_ / 2 + max_rows_ + 1) + 2 * max_rows_ + 8;
        plan_host_.resize(static_cast<size_t>(ring_));
        plan_dev_.resize(static_cast<size_t>(ring_));
        it_end_.resize(static_cast<size_t>(ring_));
        att_beg_.resize(static_cast<size_t>(ring_));
        att_end_.resize(static_cast<size_t>(ring_));
        slot_timed_.assign(static_cast<size_t>(ring_), 0);
        ts_dev_.resize(static_cast<size_t>(ring_));
        ts_host_.resize(static_cast<size_t>(2 * workers_));
        for (int i = 0; i < ring_; ++i) {
            ASV_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&plan_host_[static_cast<size_t>(i)]),
                                   static_cast<size_t>(plan_cap_) * 4, cudaHostAllocDefault));
            ASV_CUDA(cudaMalloc(&plan_dev_[static_cast<size_t>(i)], static_cast<size_t>(plan_cap_) * 4));
            ASV_CUDA(cudaEventCreateWithFlags(&it_end_[static_cast<size_t>(i)], cudaEventDisableTiming));
            ASV_CUDA(cudaEventCreate(&att_beg_[static_cast<size_t>(i)]));
            ASV_CUDA(cudaEventCreate(&att_end_[static_cast<size_t>(i)]));
            ASV_CUDA(cudaMalloc(&ts_dev_[static_cast<size_t>(i)], static_cast<size_t>(workers_) * 16));
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
    }

    ~GpuExecutor() override {
        cudaSetDevice(o_.decode_device);
        cudaDeviceSynchronize();
        if (pair_) {
            cudaSetDevice(o_.prefetch_device);
            cudaDeviceSynchronize();
            cudaSetDevice(o_.decode_device);
        }
        for (auto p : plan_host_) cudaFreeHost(p);
        for (auto p : plan_dev_) cudaFree(p);
        for (auto e : it_end_) cudaEventDestroy(e);
        for (auto e : att_beg_) cudaEventDestroy(e);
        for (auto e : att_end_) cudaEventDestroy(e);
        for (auto p : ts_dev_) cudaFree(p);
        for (auto& pr : copy_timers_) {
            cudaEventDestroy(pr.a);
            cudaEventDestroy(pr.b);
        }
        cudaEventDestroy(win_beg_);
        cudaEventDestroy(win_end_);
        cudaFree(q_);
        cudaFree(out_);
        cudaFree(k_new_);
        cudaFree(v_new_);
        cudaFree(ws_);
        if (arena_) cudaFreeHost(arena_);
        cudaStreamDestroy(compute_);
        cudaStreamDestroy(p2p_);
        cudaStreamDestroy(xfer_);
        cudaStreamDestroy(d2h_);
        cudaStreamDestroy(urgent_);
    }

    // ---------------------------------------------------------- observer
    void on_action(const prefixsim::ActionRecord& a) override {
        const auto t0 = clock_now();
        const std::string& act = a.action;
        if (act == "batch") {
            pending_batch_.push_back(a.request_id);
        } else if (act == "release") {
            ReqKV& r = kv(a.request_id);
            release_pages(r);
        } else if (act == "admit" && a.from == "wait_queue" && !admit_moved_) {
            // merged-instance FCFS: the prompt is processed in place on the decode GPU
            ReqKV& r = kv(a.request_id);
            if (r.pages.empty()) {
                r.prefix = a.blocks * 16;  // only the page count matters for the prompt's KV
                for (int64_t i = 0; i < a.blocks; ++i) r.pages.push_back(dec_.alloc());
                r.where = ReqKV::kDecode;
            }
        }
        admit_moved_ = false;
        host_ms_ += ms_since(t0);
    }

    void on_transfer(const prefixsim::TransferRecord& t) override {
        const auto t0 = clock_now();
        const int k = xfer_kind(t.kind);
        if (k >= 0) {
            stats_.logical_bytes[k] += t.bytes;
            stats_.logical_count[k] += 1;
        }
        if (!copies_active()) {
            // outside the executed span: keep the page bookkeeping, move nothing
            bookkeep_transfer(k, t);
            pending_batch_.clear();
            host_ms_ += ms_since(t0);
            return;
        }
        switch (k) {
            case ASV_XFER_BATCH_PREFETCH: {
                begin_xfer_group();
                for (const auto id : pending_batch_) fetch_from_host(id, staging_pool());
                pending_batch_.clear();
                end_xfer_group();
                break;
            }
            case ASV_XFER_STRAY_PREFETCH:
                begin_xfer_group(Lane::kUrgent);
                fetch_from_host(t.request_id, staging_pool());
                end_xfer_group();
                break;
            case ASV_XFER_ADMIT:
                if (!aligned_) {
                    // FCFS swap-in / disaggregated admit: host pool -> decode pages (PCIe)
                    begin_xfer_group(Lane::kUrgent);
                    fetch_from_host(t.request_id, &dec_);
                    end_xfer_group();
                } else {
                    admit_to_decode(t.request_id);  // candidate buffer -> running (NVLink / in place)
                }
                admit_moved_ = true;
                break;
            case ASV_XFER_EVICT:
                if (!aligned_) {
                    begin_xfer_group(Lane::kD2H);
                    write_back_to_host(t.request_id);
                    end_xfer_group();
                } else {
                    evict_to_prefetch(t.request_id);
                }
                break;
            case ASV_XFER_SPILL:
            case ASV_XFER_FLUSH:
                begin_xfer_group(Lane::kD2H);
                write_back_to_host(t.request_id);
                end_xfer_group();
                break;
            default:
                break;  // prefill_offload: prefill is off the decode path (its KV lands in the pool)
        }
        host_ms_ += ms_since(t0);
    }

    void on_iteration(const prefixsim::IterationRecord& rec, const std::vector<prefixsim::RunningMember>& running) override {
        const auto t0 = clock_now();
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
        const size_t slot = static_cast<size_t>(e % ring_);
        // throttle: the slot's previous iteration must be complete before reuse
        if (e >= ring_) retire(slot);
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
                                indices_.data(), workers_, plan_host_[slot], plan_cap_, &plan) != ASV_OK) {
            throw std::runtime_error(asv_last_error());
        }
        if (plan.total_splits > ws_splits_) throw std::runtime_error("attention workspace too small");
        ASV_CUDA(cudaSetDevice(o_.decode_device));
        if (timed && !window_open_) {
            ASV_CUDA(cudaEventRecord(win_beg_, compute_));
            window_open_ = true;
        }
        // admitted requests whose KV is still in flight: the iteration waits for it
        for (const auto& m : running) {
            ReqKV& r = kv(m.id);
            if (r.ready != nullptr) {
                ASV_CUDA(cudaStreamWaitEvent(compute_, r.ready, 0));
                r.ready = nullptr;
            }
        }
        ASV_CUDA(cudaMemcpyAsync(plan_dev_[slot], plan_host_[slot], static_cast<size_t>(plan.total_int32) * 4,
                                 cudaMemcpyHostToDevice, compute_));
        ASV_CUDA(cudaEventRecord(att_beg_[slot], compute_));
        asv_attn_args args{};
        args.q = q_;
        args.kv_pool = dec_.base();
        args.pool_pages = dec_.size();
        args.plan_dev = plan_dev_[slot];
        args.plan = &plan;
        args.k_new = k_new_;
        args.v_new = v_new_;
        args.out = out_;
        args.lse = nullptr;
        args.workspace = ws_;
        args.workspace_bytes = ws_bytes_;
        args.sm_scale = 0.08838834764831845f;
        args.pdl = o_.pdl;
        for (int l = 0; l < o_.num_layers; ++l) {
            args.layer = l;
            args.launch_index = launches_++;
            args.warp_timestamps = (timed && l == 0) ? ts_dev_[slot] : nullptr;
            if (asv_decode_attention(&shape_, &args, compute_) != ASV_OK) throw CudaError(asv_last_error());
        }
        ASV_CUDA(cudaEventRecord(att_end_[slot], compute_));
        ASV_CUDA(cudaEventRecord(it_end_[slot], compute_));
        last_it_end_ = it_end_[slot];
        slot_timed_[slot] = timed ? 1 : 0;
        if (timed) {
            ++stats_.iterations_timed;
            stats_.tokens_timed += static_cast<int64_t>(running.size());
            stats_.attn_launches += o_.num_layers;
            stats_.kernel_launches_timed += o_.num_layers * (plan.n_merge > 0 ? 2 : 1);
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
        }
        host_ms_ += ms_since(t0);
    }

    void finish(const prefixsim::MetricsLog& log, asv_engine_stats* out) {
        ASV_CUDA(cudaSetDevice(o_.decode_device));
        if (window_open_) ASV_CUDA(cudaEventRecord(win_end_, compute_));
        ASV_CUDA(cudaStreamSynchronize(compute_));
        ASV_CUDA(cudaSetDevice(xfer_device()));
        ASV_CUDA(cudaStreamSynchronize(xfer_));
        ASV_CUDA(cudaStreamSynchronize(d2h_));
        ASV_CUDA(cudaStreamSynchronize(urgent_));
        ASV_CUDA(cudaSetDevice(o_.decode_device));
        ASV_CUDA(cudaStreamSynchronize(p2p_));
        for (int64_t e = std::max<int64_t>(0, executed_ - ring_); e < executed_; ++e) retire(static_cast<size_t>(e % ring_));
        if (window_open_) {
            float ms = 0.f;
            ASV_CUDA(cudaEventElapsedTime(&ms, win_beg_, win_end_));
            stats_.window_ms = ms;
        }
        for (auto& pr : copy_timers_) {
            float ms = 0.f;
            if (cudaEventElapsedTime(&ms, pr.a, pr.b) == cudaSuccess) {
                (pr.p2p ? stats_.p2p_busy_ms : stats_.h2d_busy_ms) += ms;
            }
        }
        stats_.iterations_total = iterations_total_;
        stats_.measured_idle_frac = span_ns_ > 0 ? 1.0 - busy_ns_ / span_ns_ : 0.0;
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

    // page ownership changes of a transfer whose bytes are not moved
    void bookkeep_transfer(int k, const prefixsim::TransferRecord& t) {
        switch (k) {
            case ASV_XFER_BATCH_PREFETCH:
                for (const auto id : pending_batch_) fetch_from_host(id, staging_pool());
                break;
            case ASV_XFER_STRAY_PREFETCH: fetch_from_host(t.request_id, staging_pool()); break;
            case ASV_XFER_ADMIT:
                if (!aligned_) fetch_from_host(t.request_id, &dec_);
                else admit_to_decode(t.request_id);
                admit_moved_ = true;
                break;
            case ASV_XFER_EVICT:
                if (!aligned_) write_back_to_host(t.request_id);
                else evict_to_prefetch(t.request_id);
                break;
            case ASV_XFER_SPILL:
            case ASV_XFER_FLUSH: write_back_to_host(t.request_id); break;
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

    // group copies issued by one decision so one event pair times them
    // Batch prefetches run on xfer_, small urgent H2D moves (strays, swap-ins) on
    // urgent_ so they never queue behind a whole batch, D2H on d2h_ (both PCIe
    // directions at once).
    enum class Lane { kBulk, kUrgent, kD2H };
    void begin_xfer_group(Lane lane_sel = Lane::kBulk) {
        group_timed_ = copies_active() && in_window();
        cur_ = lane_sel == Lane::kD2H ? d2h_ : (lane_sel == Lane::kUrgent ? urgent_ : xfer_);
        cur_ev_ = lane_sel == Lane::kD2H ? &d2h_ev_ : (lane_sel == Lane::kUrgent ? &urgent_ev_ : &xfer_ev_);
        if (!copies_active()) return;
        ASV_CUDA(cudaSetDevice(xfer_device()));
        // pages written/read below may have been used by the last launched iteration
        cudaEvent_t& waited = lane_sel == Lane::kD2H ? waited_it_end_d2h_
                              : (lane_sel == Lane::kUrgent ? waited_it_end_urg_ : waited_it_end_);
        if (last_it_end_ != nullptr && waited != last_it_end_) {
            ASV_CUDA(cudaStreamWaitEvent(cur_, last_it_end_, 0));
            waited = last_it_end_;
        }
        if (group_timed_) {
            CopyTimer t{};
            ASV_CUDA(cudaEventCreate(&t.a));
            ASV_CUDA(cudaEventCreate(&t.b));
            ASV_CUDA(cudaEventRecord(t.a, cur_));
            copy_timers_.push_back(t);
        }
    }
    cudaEvent_t end_xfer_group() {
        if (!copies_active()) return nullptr;
        if (group_timed_) ASV_CUDA(cudaEventRecord(copy_timers_.back().b, cur_));
        cudaEvent_t ev = cur_ev_->record(cur_);
        for (auto id : group_ready_) kv(id).ready = ev;
        group_ready_.clear();
        for (auto& q : group_quarantine_) q.first->release_after(ev, std::move(q.second));
        group_quarantine_.clear();
        ASV_CUDA(cudaSetDevice(o_.decode_device));
        return ev;
    }

    char* host_page(prefixsim::RequestId id, int64_t j) const {
        const int64_t a = (id * 7919 + j) % arena_pages_;
        return arena_ + a * page_bytes_;
    }

    // copy `tokens` tokens of KV between host pages and device pages (exact bytes)
    // KV moves go through the C-ABI copy routines (kv_copy.cpp): whole pages as
    // 2-D copies, the valid rows of a partial last page as one 3-D copy.
    int64_t copy_kv(const std::vector<int32_t>& pages, const PagePool& pool, prefixsim::RequestId id, int64_t tokens,
                    bool to_device) {
        host_ptrs_.clear();
        for (int64_t j = 0; j < (tokens + 15) / 16; ++j) host_ptrs_.push_back(host_page(id, j));
        int64_t moved = 0;
        const int rc = to_device ? asv_kv_copy_h2d(&shape_, pool.base(), pool.size(), pages.data(), tokens,
                                                   host_ptrs_.data(), cur_, &moved)
                                 : asv_kv_copy_d2h(&shape_, pool.base(), pool.size(), pages.data(), tokens,
                                                   const_cast<void* const*>(host_ptrs_.data()), cur_, &moved);
        if (rc != ASV_OK) throw CudaError(asv_last_error());
        return moved;
    }

    void fetch_from_host(prefixsim::RequestId id, PagePool* pool) {
        ReqKV& r = kv(id);
        const prefixsim::Request& q = (*requests_)[static_cast<std::size_t>(id)];
        r.prefix = q.prefix_len;
        release_pages(r);  // (defensive) a request never holds pages while pooled
        const int64_t n = (q.prefix_len + 15) / 16;
        for (int64_t j = 0; j < n; ++j) r.pages.push_back(pool->alloc());
        r.where = pool == &dec_ ? ReqKV::kDecode : ReqKV::kPrefetch;
        if (!copies_active()) return;
        const int64_t moved = copy_kv(r.pages, *pool, id, q.prefix_len, true);
        stats_.h2d_bytes += moved;
        if (group_timed_) stats_.h2d_bytes_window += moved;
        r.ready = cur_ev_->record(cur_);  // this request is usable as soon as its own pages land
    }

    void write_back_to_host(prefixsim::RequestId id) {
        ReqKV& r = kv(id);
        const prefixsim::Request& q = (*requests_)[static_cast<std::size_t>(id)];
        PagePool* pool = r.where == ReqKV::kPrefetch ? &pre_ : &dec_;
        if (copies_active() && !r.pages.empty()) {
            if (r.ready != nullptr) {
                ASV_CUDA(cudaStreamWaitEvent(cur_, r.ready, 0));
                r.ready = nullptr;
            }
            const int64_t moved = copy_kv(r.pages, *pool, id, q.prefix_len, false);
            stats_.d2h_bytes += moved;
            if (group_timed_) stats_.d2h_bytes_window += moved;
            group_quarantine_.push_back({pool, std::move(r.pages)});
            r.pages.clear();
        } else {
            pool->release(r.pages);
            r.pages.clear();
        }
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
        for (size_t j = 0; j < r.pages.size(); ++j) dst.push_back(dec_.alloc());
        if (copies_active()) {
            ASV_CUDA(cudaSetDevice(o_.decode_device));
            if (r.ready != nullptr) ASV_CUDA(cudaStreamWaitEvent(p2p_, r.ready, 0));
            if (last_it_end_ != nullptr) ASV_CUDA(cudaStreamWaitEvent(p2p_, last_it_end_, 0));
            CopyTimer t{};
            const bool timed = in_window();
            if (timed) {
                ASV_CUDA(cudaEventCreate(&t.a));
                ASV_CUDA(cudaEventCreate(&t.b));
                t.p2p = true;
                ASV_CUDA(cudaEventRecord(t.a, p2p_));
            }
            const int64_t moved = copy_peer(dst, dec_, r.pages, pre_, (*requests_)[static_cast<std::size_t>(id)].prefix_len);
            stats_.p2p_bytes += moved;
            if (timed) {
                ASV_CUDA(cudaEventRecord(t.b, p2p_));
                copy_timers_.push_back(t);
                stats_.p2p_bytes_window += moved;
            }
            cudaEvent_t ev = p2p_ev_.record(p2p_);
            pre_.release_after(ev, std::move(r.pages));
            r.ready = ev;
        } else {
            pre_.release(r.pages);
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
            ASV_CUDA(cudaSetDevice(o_.decode_device));
            if (last_it_end_ != nullptr) ASV_CUDA(cudaStreamWaitEvent(p2p_, last_it_end_, 0));
            const int64_t moved = copy_peer(dst, pre_, r.pages, dec_, (*requests_)[static_cast<std::size_t>(id)].prefix_len);
            stats_.p2p_bytes += moved;
            if (in_window()) stats_.p2p_bytes_window += moved;
            cudaEvent_t ev = p2p_ev_.record(p2p_);
            dec_.release_after(ev, std::move(r.pages));
            r.ready = ev;
        } else {
            dec_.release(r.pages);
        }
        r.pages = std::move(dst);
        r.where = ReqKV::kPrefetch;
    }

    int64_t copy_peer(const std::vector<int32_t>& dst, const PagePool& dpool, const std::vector<int32_t>& src,
                      const PagePool& spool, int64_t tokens) {
        int64_t moved = 0;
        if (asv_kv_copy_d2d(&shape_, dpool.base(), dpool.size(), dpool.device(), dst.data(), spool.base(), spool.size(),
                            spool.device(), src.data(), tokens, p2p_, &moved) != ASV_OK) {
            throw CudaError(asv_last_error());
        }
        return moved;
    }

    void release_pages(ReqKV& r) {
        if (r.pages.empty()) return;
        (r.where == ReqKV::kPrefetch ? pre_ : dec_).release(r.pages);
        r.pages.clear();
        r.ready = nullptr;
        r.where = ReqKV::kHost;
    }

    void retire(size_t slot) {
        ASV_CUDA(cudaEventSynchronize(it_end_[slot]));
        if (slot_timed_[slot]) {
            float ms = 0.f;
            ASV_CUDA(cudaEventElapsedTime(&ms, att_beg_[slot], att_end_[slot]));
            stats_.attn_ms += ms;
            slot_timed_[slot] = 0;
            // measured bubble of the layer-0 launch: idle warp time inside its span
            ASV_CUDA(cudaMemcpy(ts_host_.data(), ts_dev_[slot], ts_host_.size() * 8, cudaMemcpyDeviceToHost));
            uint64_t lo = UINT64_MAX, hi = 0;
            double busy = 0.0;
            for (int32_t w = 0; w < workers_; ++w) {
                const uint64_t a = ts_host_[2 * w], b = ts_host_[2 * w + 1];
                if (b <= a) continue;
                lo = std::min(lo, a);
                hi = std::max(hi, b);
                busy += static_cast<double>(b - a);
            }
            if (hi > lo) {
                const double span = static_cast<double>(hi - lo) * workers_;
                busy_ns_ += busy;
                span_ns_ += span;
                stats_.measured_bubble_ms += (span - busy) / workers_ * 1e-6 * o_.num_layers;
            }
        }
        dec_.reclaim(false);
        if (pair_) pre_.reclaim(false);
    }

 public:
    const std::vector<prefixsim::Request>* requests_ = nullptr;

 private:
    struct CopyTimer {
        cudaEvent_t a = nullptr, b = nullptr;
        bool p2p = false;
    };
    asv_engine_opts o_;
    asv_attn_shape shape_{};
    int64_t page_bytes_ = 0, row_bytes_all_ = 0, slice_ = 0;
    bool pair_ = false;
    int64_t dec_pages_ = 0, pre_pages_ = 0;
    PagePool dec_, pre_;
    cudaStream_t compute_ = nullptr, p2p_ = nullptr, xfer_ = nullptr, d2h_ = nullptr, urgent_ = nullptr,
                 cur_ = nullptr;
    EventRing xfer_ev_, d2h_ev_, urgent_ev_, p2p_ev_;
    EventRing* cur_ev_ = nullptr;
    cudaEvent_t waited_it_end_d2h_ = nullptr, waited_it_end_urg_ = nullptr;
    char* arena_ = nullptr;
    int64_t arena_pages_ = 1;
    int32_t workers_ = 0;
    int64_t max_rows_ = 0;
    void *q_ = nullptr, *out_ = nullptr, *k_new_ = nullptr, *v_new_ = nullptr, *ws_ = nullptr;
    size_t ws_bytes_ = 0;
    int32_t ws_splits_ = 0;
    int ring_ = 16;
    int64_t plan_cap_ = 0;
    std::vector<int32_t*> plan_host_, plan_dev_;
    std::vector<cudaEvent_t> it_end_, att_beg_, att_end_;
    std::vector<int> slot_timed_;
    cudaEvent_t last_it_end_ = nullptr, waited_it_end_ = nullptr;
    cudaEvent_t win_beg_ = nullptr, win_end_ = nullptr;
    bool window_open_ = false, last_timed_end_ = false, group_timed_ = false, admit_moved_ = false;
    std::vector<ReqKV> reqs_;
    std::vector<prefixsim::RequestId> pending_batch_;
    std::vector<prefixsim::RequestId> group_ready_;
    std::vector<std::pair<PagePool*, std::vector<int32_t>>> group_quarantine_;
    std::vector<CopyTimer> copy_timers_;
    std::vector<int32_t> seq_, indptr_, indices_;
    std::vector<const void*> host_ptrs_;
    int64_t executed_ = 0, iterations_total_ = 0;
    uint32_t launches_ = 0;
    double host_ms_ = 0.0;
    double first_timed_start_ = -1.0, last_timed_end_ms_ = 0.0;
    std::vector<uint64_t*> ts_dev_;
    std::vector<uint64_t> ts_host_;
    double busy_ns_ = 0.0, span_ns_ = 0.0;
    asv_engine_stats stats_{};
};

}  // namespace

int engine_run(const char* config_json, const char* policy_override, const asv_engine_opts* opts,
               asv_engine_stats* stats) {
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
        prefixsim::Simulation sim(cfg.sim, model, reqs);
        GpuExecutor ex(*opts, cfg.sim, model.spec, reqs.size());
        ex.requests_ = &sim.requests();
        ex.aligned_ = cfg.sim.policy == prefixsim::Policy::kAligned;
        sim.set_observer(&ex);
        const auto t0 = std::chrono::steady_clock::now();
        prefixsim::MetricsLog log = sim.run();
        (void)t0;
        ex.finish(log, stats);
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
    return asv::engine_run(config_json, policy_override, opts, stats);
}
