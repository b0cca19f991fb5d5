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

// Layer-major device pools are split into equal page GROUPS so that the layer
// pitch of a group (group_pages * slice) stays below 2 GiB: the copy engines
// run a 2-D copy at full PCIe rate only below that pitch (measured on B200:
// 54 GB/s at a 1 GiB pitch, 29.7 GB/s = one row per copy at >= 2 GiB;
// tools/copy_tlb_probe.py).  Group g holds pages [g*G, (g+1)*G) as
// [L][G][slice]; page p's layer-l slice is at slice index
//   pool_slot(p) + l*G,  pool_slot(p) = p + (p / G) * G * (L - 1).
// A pool that fits one group (every test-sized pool) is plain [L][pages][slice].
constexpr int64_t kMaxGroupPitch = (int64_t(1) << 31) - 1;

inline int64_t pool_group_pages(int64_t slice, int64_t pool_pages) {
    const int64_t gmax = kMaxGroupPitch / slice;
    const int64_t groups = (pool_pages + gmax - 1) / gmax;
    return pool_pages / groups;
}
inline int64_t pool_usable_pages(int64_t slice, int64_t pool_pages) {
    const int64_t g = pool_group_pages(slice, pool_pages);
    return (pool_pages / g) * g;
}
inline int64_t pool_slot(int64_t page, int64_t group_pages, int64_t layers) {
    return page + (page / group_pages) * group_pages * (layers - 1);
}

// Launch description for the decode-attention kernel (decode_attn.cu).
struct AttnLaunch {
    int group;              // n_q / n_kv
    int grid;               // persistent CTAs
    bool pdl;               // programmatic dependent launch
    bool f16;               // KV / q / out element type: fp16 (else bf16)
    const void* q;
    void* pool;
    int64_t page_bytes;     // one layer slice of one page (pool_slot unit)
    int64_t layer_off;      // layer * group_pages * page_bytes
    int64_t v_off;
    int32_t group_pages;    // pages per layer-major group (pool_group_pages)
    int32_t group_skip;     // group_pages * (L - 1): pool_slot(p) = p + (p / group_pages) * group_skip
    int32_t usable_pages;   // page ids must be < this (the kernel traps otherwise)
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
    uint32_t* work;           // 2 counters of this launch parity
    const int32_t* merge_reqs;  // requests with > 1 split (merge kernel rows)
    int32_t n_merge;
    int sms;
    float sm_scale;
    unsigned long long* warp_ts;  // optional per-warp %globaltimer (start, end)
    bool defer_merge;             // leave this launch's partials to the next launch (no merge kernel)
    const float* prev_part_o;     // previous launch's deferred partials (other parity), or null
    const float* prev_part_ml;
    void* prev_out;               // non-null: merge the previous launch's split rows into it
    float* prev_lse;
    int32_t warm_items;           // > 0: L2-warm mode — only prefetch the first warm_pages pages of the
    int32_t warm_pages;           //       first warm_items work items into L2 (no attention, no merge)
};

int attn_warps_per_cta(int group, bool f16 = false);
cudaError_t attn_occupancy(int group, int* blocks_per_sm);
cudaError_t attn_launch(const AttnLaunch& a, cudaStream_t st);
// n_int32 rounded up to a multiple of 4 (16-byte units); both pointers 16-byte aligned
cudaError_t sm_copy(const int32_t* src, int32_t* dst, int64_t n_int32, cudaStream_t st);
// per attention launch l: out[3l..3l+2] = (first warp start, last warp end, summed warp busy) of the
// launch's per-warp %globaltimer pairs ts[l][workers][2], which it zeroes (measured bubble)
cudaError_t warp_span_reduce(uint64_t* ts, int32_t workers, int32_t launches, uint64_t* out, cudaStream_t st);

// device-to-device KV page moves on the SMs (kv_move.cu): pages per launch (kernel parameter arrays)
constexpr int kMoveChunk = 1024;
cudaError_t kv_move_launch(const void* src_pool, int64_t src_gp, void* dst_pool, int64_t dst_gp, int64_t slice,
                           int32_t layers, const int32_t* src_pages, const int32_t* dst_pages, int64_t tokens,
                           cudaStream_t st);
cudaError_t kv_move_preload();

// decode-step linear layers (decode_gemm.cu)
cudaError_t linear_preload();
cudaError_t linear_chain_preload();
cudaError_t rmsnorm_launch(const void* h, const void* gamma, void* out, int dim, int batch, int rows_out, float eps,
                           bool pdl, cudaStream_t st);
cudaError_t rmsnorm_preload();
cudaError_t fill_random_bf16(void* p, int64_t n, uint64_t seed, float scale, float offset, cudaStream_t st);

// thread-local last error (asv_last_error)
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

}  // namespace asv
