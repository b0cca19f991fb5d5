// Host runtime pieces of the KV-move path (not part of the ABI).
//
//  * SeqFlags — cross-stream ordering by 32-bit sequence values in mapped
//    pinned host memory, written and awaited BY THE STREAMS
//    (cuStreamWriteValue32 / cuStreamWaitValue32, GEQ with wrap-around).
//    Unlike cudaStreamWaitEvent, a wait can be enqueued before the matching
//    write has been issued, so the thread that launches decode iterations and
//    the thread that issues KV copies never wait for each other.
//  * CopyWorker — one host thread that issues every copy-stream operation.
//    Enqueuing a copy can block inside the driver once a stream's queue is full
//    (measured: 100 us per 8 MiB page copy with multi-GB batch prefetches in
//    flight, 1.3 us when idle); on its own thread that back-pressure never
//    stalls the launch of decode iterations.
//  * Serial mode (ASV_SERIAL=1, or automatically under a CUDA profiler /
//    sanitizer injection): every posted operation runs inline on the posting
//    thread and each flag write synchronises its stream and then sets the flag
//    from the host; a flag wait is a host-side check (never a stream wait).  A
//    profiler that serialises kernels across streams (Nsight Compute) would
//    otherwise park a stream on a flag whose writer it never schedules.
#pragma once

#include <nvtx3/nvToolsExt.h>  // header-only NVTX: a named range per posted operation (Nsight timelines)

#include <cuda.h>
#include <cuda_runtime.h>

#include <atomic>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <functional>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>

namespace asv {

// ASV_SERIAL=1, or a CUDA injection library (ncu / nsys / compute-sanitizer) is loaded.  Nsight
// Compute starts its target through an LD_PRELOAD launcher and does not leave CUDA_INJECTION64_PATH
// in the environment (measured), so the process's own mappings are checked too.
inline bool serial_mode_requested() {
    if (const char* e = std::getenv("ASV_SERIAL")) return std::atoi(e) != 0;
    if (std::getenv("CUDA_INJECTION64_PATH") != nullptr) return true;
    if (const char* pre = std::getenv("LD_PRELOAD")) {
        const std::string s(pre);
        if (s.find("TreeLauncher") != std::string::npos || s.find("nsight") != std::string::npos) return true;
    }
    std::FILE* f = std::fopen("/proc/self/maps", "r");
    if (f == nullptr) return false;
    char line[4096];
    bool hit = false;
    while (!hit && std::fgets(line, sizeof(line), f) != nullptr) {
        hit = std::strstr(line, "cuda-injection") != nullptr || std::strstr(line, "InjectionTarget") != nullptr ||
              std::strstr(line, "TreeLauncher") != nullptr || std::strstr(line, "libToolsInjection") != nullptr ||
              std::strstr(line, "sanitizer-public") != nullptr || std::strstr(line, "libsanitizer-collection") != nullptr;
    }
    std::fclose(f);
    return hit;
}

class SeqFlags {
 public:
    static constexpr int kSlots = 8;
    void set_serial(bool on) { serial_ = on; }
    bool serial() const { return serial_; }

    void init() {
        if (cudaHostAlloc(reinterpret_cast<void**>(&host_), kSlots * sizeof(uint32_t),
                          cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
            throw std::runtime_error("SeqFlags: cudaHostAlloc failed");
        }
        for (int i = 0; i < kSlots; ++i) host_[i] = 0;
        void* d = nullptr;
        if (cudaHostGetDevicePointer(&d, host_, 0) != cudaSuccess) throw std::runtime_error("SeqFlags: no device map");
        dev_ = reinterpret_cast<CUdeviceptr>(d);
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuStreamWaitValue32", reinterpret_cast<void**>(&wait_), cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess ||
            cudaGetDriverEntryPoint("cuStreamWriteValue32", reinterpret_cast<void**>(&write_), cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            throw std::runtime_error("SeqFlags: stream memory operations unavailable");
        }
    }
    ~SeqFlags() {
        if (host_ != nullptr) cudaFreeHost(host_);
    }
    // `st` waits until flag[slot] >= v (cyclic 32-bit compare)
    void wait(cudaStream_t st, int slot, uint32_t v) const {
        if (serial_) {  // everything before this point has completed (program order + stream syncs)
            if (!reached(slot, v))
                throw std::logic_error("serial mode: wait on sequence flag " + std::to_string(slot) + " >= " +
                                       std::to_string(v) + " that no earlier operation writes");
            return;
        }
        check(wait_(reinterpret_cast<CUstream>(st), dev_ + slot * sizeof(uint32_t), v, CU_STREAM_WAIT_VALUE_GEQ),
              "cuStreamWaitValue32");
    }
    // `st` sets flag[slot] = v once its prior work is complete
    void write(cudaStream_t st, int slot, uint32_t v) const {
        if (serial_) {
            if (cudaStreamSynchronize(st) != cudaSuccess) throw std::runtime_error("serial mode: stream sync failed");
            reinterpret_cast<volatile uint32_t*>(host_)[slot] = v;
            return;
        }
        check(write_(reinterpret_cast<CUstream>(st), dev_ + slot * sizeof(uint32_t), v, CU_STREAM_WRITE_VALUE_DEFAULT),
              "cuStreamWriteValue32");
    }
    uint32_t value(int slot) const { return reinterpret_cast<volatile uint32_t*>(host_)[slot]; }
    bool reached(int slot, uint32_t v) const {
        const uint32_t cur = reinterpret_cast<volatile uint32_t*>(host_)[slot];
        return static_cast<int32_t>(cur - v) >= 0;
    }
    // host override (error paths): release every wait up to v
    void force(int slot, uint32_t v) { reinterpret_cast<volatile uint32_t*>(host_)[slot] = v; }

 private:
    static void check(CUresult r, const char* what) {
        if (r != CUDA_SUCCESS) throw std::runtime_error(std::string(what) + " failed (" + std::to_string(r) + ")");
    }
    using Fn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
    uint32_t* host_ = nullptr;
    CUdeviceptr dev_ = 0;
    Fn wait_ = nullptr, write_ = nullptr;
    bool serial_ = false;
};

class CopyWorker {
 public:
    // inline: post() runs the operation on the calling thread (serial mode), no worker thread
    void start(bool inline_ops = false) {
        inline_ = inline_ops;
        if (!inline_) th_ = std::thread([this] { loop(); });
    }
    void post(std::function<void()> fn, const char* label = "op") {
        if (inline_) {
            cur_.store(label);
            nvtxRangePushA(label);
            fn();  // exceptions propagate to the caller
            nvtxRangePop();
            done_.fetch_add(1);
            return;
        }
        {
            std::lock_guard<std::mutex> lk(m_);
            q_.push_back({std::move(fn), label});
        }
        cv_.notify_one();
    }
    const char* current() const { return cur_.load(); }
    // block until everything posted so far has been issued
    void drain() {
        std::unique_lock<std::mutex> lk(m_);
        idle_.wait(lk, [&] { return q_.empty() && !busy_; });
    }
    // skip whatever is still queued (error paths), then join
    void stop(bool abandon) {
        {
            std::lock_guard<std::mutex> lk(m_);
            stop_ = true;
            if (abandon) q_.clear();
        }
        cv_.notify_one();
        if (th_.joinable()) th_.join();
    }
    bool failed() const { return failed_.load(); }
    // debugging: closures completed / queued
    uint64_t done() const { return done_.load(); }
    size_t queued() {
        std::lock_guard<std::mutex> lk(m_);
        return q_.size();
    }
    std::string error() {
        std::lock_guard<std::mutex> lk(m_);
        return err_;
    }
    ~CopyWorker() { stop(true); }

 private:
    void loop() {
        for (;;) {
            std::function<void()> fn;
            {
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [&] { return stop_ || !q_.empty(); });
                if (q_.empty()) return;  // stop requested and drained
                fn = std::move(q_.front().first);
                cur_.store(q_.front().second);
                q_.pop_front();
                busy_ = true;
            }
            if (!failed_.load()) {
                nvtxRangePushA(cur_.load());
                try {
                    fn();
                    nvtxRangePop();
                } catch (const std::exception& e) {
                    nvtxRangePop();
                    std::lock_guard<std::mutex> lk(m_);
                    err_ = e.what();
                    failed_.store(true);
                }
            }
            done_.fetch_add(1);
            {
                std::lock_guard<std::mutex> lk(m_);
                busy_ = false;
                if (q_.empty()) idle_.notify_all();
            }
        }
    }
    std::mutex m_;
    std::condition_variable cv_, idle_;
    std::deque<std::pair<std::function<void()>, const char*>> q_;
    std::atomic<const char*> cur_{""};
    bool stop_ = false, busy_ = false;
    std::atomic<bool> failed_{false};
    std::atomic<uint64_t> done_{0};
    std::string err_;
    std::thread th_;
    bool inline_ = false;
};

}  // namespace asv
