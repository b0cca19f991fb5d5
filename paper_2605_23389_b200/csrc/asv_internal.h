// Internal glue between the C ABI (include/asv.h), the host runtime and the
// CUDA kernels.  Not part of the ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace asv {

// Launch description for the decode-attention kernel (decode_attn.cu).
struct AttnLaunch {
    int group;              // n_q / n_kv
    int grid;               // persistent CTAs
    const void* q;
    void* pool;
    int64_t page_bytes;
    int64_t layer_off;
    int64_t v_off;
    const int32_t* seq_lens;
    const int32_t* page_indptr;
    const int32_t* page_indices;
    const int32_t* split_indptr;
    const int32_t* item_tab;  // int2 pairs
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
    float sm_scale;
};

int attn_warps_per_cta();
cudaError_t attn_occupancy(int group, int* blocks_per_sm);
cudaError_t attn_launch(const AttnLaunch& a, cudaStream_t st);

// thread-local last error (asv_last_error)
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

}  // namespace asv
