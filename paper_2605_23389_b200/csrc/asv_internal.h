// Internal glue between the C ABI (include/asv.h), the host runtime and the
// CUDA kernels.  Not part of the ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace asv {

// Words per split descriptor in the plan buffer (decode_attn.cu Desc):
// [r, slot, page_begin, page_end, seq_len, nsplit, append_phys, 0] + 32 page ids.
constexpr int kDescWords = 40;
constexpr int kMaxItemPages = 32;

// Launch description for the decode-attention kernel (decode_attn.cu).
struct AttnLaunch {
    int group;              // n_q / n_kv
    int grid;               // persistent CTAs
    bool pdl;               // programmatic dependent launch
    const void* q;
    void* pool;
    int64_t page_bytes;
    int64_t layer_off;
    int64_t v_off;
    const int32_t* gdesc;
    const int32_t* split_base;
    int32_t num_items;
    int32_t n_kv;
    int32_t n_q;
    const void* k_new;
    const void* v_new;
    void* out;
    float* lse;
    float* part_o;
    float* part_ml;           // float2 pairs
    int32_t* sem;
    uint32_t* work;           // 2 counters of this launch parity
    const int32_t* merge_reqs;  // requests with > 1 split (merge kernel rows)
    int32_t n_merge;
    int sms;
    float sm_scale;
    unsigned long long* warp_ts;  // optional per-warp %globaltimer (start, end)
};

int attn_warps_per_cta(int group);
cudaError_t attn_occupancy(int group, int* blocks_per_sm);
cudaError_t attn_launch(const AttnLaunch& a, cudaStream_t st);

// thread-local last error (asv_last_error)
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

}  // namespace asv
