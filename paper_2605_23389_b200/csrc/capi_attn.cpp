// C ABI of the decode-attention operator: split-KV planning (K4, host) and the
// K1/K2/K3 launch.  See include/asv.h for the contract and the reference
// functions each entry point replaces.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/asv.h"
#include "asv_internal.h"

namespace asv {

namespace {
thread_local std::string g_last_error;
constexpr int64_t kHeadBytes = 256;  // per-parity dynamic-schedule counters; partials follow
constexpr int64_t kBlockBytes = 16 * 128 * 2;

int group_of(const asv_attn_shape* s) { return s->num_q_heads / s->num_kv_heads; }

int check_shape(const asv_attn_shape* s) {
    if (s == nullptr) return fail(ASV_ERR_INVALID, "null shape");
    if (s->head_dim != 128) return fail(ASV_ERR_INVALID, "head_dim must be 128");
    if (s->page_size != 16) return fail(ASV_ERR_INVALID, "page_size must be 16 (block_size)");
    if (s->num_kv_heads < 1 || s->num_q_heads < 1 || s->num_layers < 1)
        return fail(ASV_ERR_INVALID, "shape fields must be strictly positive");
    if (s->num_q_heads % s->num_kv_heads != 0)
        return fail(ASV_ERR_INVALID, "num_q_heads must be a multiple of num_kv_heads");
    const int g = group_of(s);
    if (g != 1 && g != 2 && g != 4 && g != 5 && g != 8)
        return fail(ASV_ERR_INVALID, "query group size must be one of 1, 2, 4, 5, 8");
    return ASV_OK;
}

struct OccCache {
    std::mutex mu;
    int dev[64][9] = {};
};
OccCache g_occ;

}  // namespace

void set_error(const std::string& msg) { g_last_error = msg; }
int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}
int cuda_fail(cudaError_t e, const char* what) {
    return fail(ASV_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace asv

using namespace asv;

extern "C" {

const char* asv_last_error(void) { return g_last_error.c_str(); }
int asv_abi_version(void) { return 2; }

int64_t asv_struct_size(const char* name) {
    if (name == nullptr) return -1;
    const std::string n(name);
    if (n == "asv_attn_shape") return static_cast<int64_t>(sizeof(asv_attn_shape));
    if (n == "asv_attn_plan") return static_cast<int64_t>(sizeof(asv_attn_plan));
    if (n == "asv_attn_args") return static_cast<int64_t>(sizeof(asv_attn_args));
    if (n == "asv_linear_args") return static_cast<int64_t>(sizeof(asv_linear_args));
    if (n == "asv_engine_opts") return static_cast<int64_t>(sizeof(asv_engine_opts));
    if (n == "asv_engine_stats") return static_cast<int64_t>(sizeof(asv_engine_stats));
    return -1;
}
void asv_free(void* p) { std::free(p); }

int64_t asv_page_bytes(const asv_attn_shape* s) {
    if (check_shape(s) != ASV_OK) return -1;
    return static_cast<int64_t>(s->num_layers) * 2 * s->num_kv_heads * kBlockBytes;
}

int64_t asv_page_offset(const asv_attn_shape* s, int32_t layer, int32_t kv, int32_t head,
                        int32_t token, int32_t dim) {
    if (check_shape(s) != ASV_OK) return -1;
    const int64_t block = ((static_cast<int64_t>(layer) * 2 + kv) * s->num_kv_heads + head) * kBlockBytes;
    const int c = dim / 8;
    return block + token * 256 + ((c ^ (token & 7)) << 4) + (dim % 8) * 2;
}

int64_t asv_pool_offset(const asv_attn_shape* s, int64_t pool_pages, int64_t page, int32_t layer, int32_t kv,
                        int32_t head, int32_t token, int32_t dim) {
    if (check_shape(s) != ASV_OK) return -1;
    const int64_t slice = static_cast<int64_t>(2) * s->num_kv_heads * kBlockBytes;
    if (pool_pages < 1 || page < 0 || page >= pool_usable_pages(slice, pool_pages)) {
        fail(ASV_ERR_INVALID, "page outside the usable pool");
        return -1;
    }
    const int64_t gp = pool_group_pages(slice, pool_pages);
    const int64_t sl = pool_slot(page, gp, s->num_layers) + static_cast<int64_t>(layer) * gp;
    const int64_t block = sl * slice + (static_cast<int64_t>(kv) * s->num_kv_heads + head) * kBlockBytes;
    const int c = dim / 8;
    return block + token * 256 + ((c ^ (token & 7)) << 4) + (dim % 8) * 2;
}

int64_t asv_pool_group_pages(const asv_attn_shape* s, int64_t pool_pages) {
    if (check_shape(s) != ASV_OK) return -1;
    if (pool_pages < 1) return fail(ASV_ERR_INVALID, "pool_pages must be >= 1"), -1;
    return pool_group_pages(static_cast<int64_t>(2) * s->num_kv_heads * kBlockBytes, pool_pages);
}

int64_t asv_pool_usable_pages(const asv_attn_shape* s, int64_t pool_pages) {
    if (check_shape(s) != ASV_OK) return -1;
    if (pool_pages < 1) return fail(ASV_ERR_INVALID, "pool_pages must be >= 1"), -1;
    return pool_usable_pages(static_cast<int64_t>(2) * s->num_kv_heads * kBlockBytes, pool_pages);
}

int asv_attn_num_workers(const asv_attn_shape* shape, int device, int32_t* workers_out) {
    if (int rc = check_shape(shape)) return rc;
    const int g = group_of(shape);
    int sms = 0;
    cudaError_t e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceGetAttribute");
    int blocks = 0;
    {
        std::lock_guard<std::mutex> lk(g_occ.mu);
        int& cached = g_occ.dev[device & 63][g];
        if (cached == 0) {
            int prev = 0;
            cudaGetDevice(&prev);
            cudaSetDevice(device);
            e = attn_occupancy(g, &cached);
            cudaSetDevice(prev);
            if (e != cudaSuccess) return cuda_fail(e, "occupancy query");
            if (cached < 1) return fail(ASV_ERR_CUDA, "decode kernel cannot be resident");
        }
        blocks = cached;
    }
    *workers_out = sms * blocks * attn_warps_per_cta(g);
    return ASV_OK;
}

int asv_attn_plan_build(const asv_attn_shape* shape, int32_t batch, const int32_t* seq_lens,
                        const int32_t* page_indptr, const int32_t* page_indices, int32_t num_workers,
                        int32_t* plan_buf, int64_t plan_cap, asv_attn_plan* plan_out) {
    if (int rc = check_shape(shape)) return rc;
    if (batch < 1) return fail(ASV_ERR_INVALID, "empty batch");
    if (num_workers < 1) return fail(ASV_ERR_INVALID, "num_workers must be >= 1");
    const int n_kv = shape->num_kv_heads;
    std::vector<int32_t> npages(static_cast<size_t>(batch));
    for (int r = 0; r < batch; ++r) {
        const int32_t s = seq_lens[r];
        if (s < 1) return fail(ASV_ERR_INVALID, "prefix lengths must be >= 1");
        const int32_t np = (s + 15) / 16;
        if (page_indptr[r + 1] - page_indptr[r] < np)
            return fail(ASV_ERR_INVALID, "page table shorter than ceil(seq_len/16) for request " +
                                             std::to_string(r));
        npages[static_cast<size_t>(r)] = np;
    }
    if (page_indptr[0] != 0) return fail(ASV_ERR_INVALID, "page_indptr[0] must be 0");

    // Split size (pages per warp item, <= 32): items are pulled dynamically in
    // longest-first order, so the makespan is ~ total/W plus about half an item
    // of tail; each item also pays a fixed cost (q load, epilogue) and each
    // split request a merge.
    const double item_overhead = 1.5, merge_cost = 0.5;
    std::vector<int32_t> best_ns(static_cast<size_t>(batch), 1), ns(static_cast<size_t>(batch));
    double best = -1.0;
    static const int kChunks[] = {2, 3, 4, 6, 8, 10, 12, 16, 20, 24, 28, 32};
    static const int forced_chunk = [] {  // ASV_PLAN_CHUNK=<pages>: tuning experiments only
        const char* e = getenv("ASV_PLAN_CHUNK");
        return e != nullptr ? atoi(e) : 0;
    }();
    for (const int c : kChunks) {
        if (forced_chunk > 0 && c != forced_chunk) continue;
        double total = 0.0;
        int max_item = 0;
        for (int r = 0; r < batch; ++r) {
            const int n = npages[static_cast<size_t>(r)];
            const int k = (n + c - 1) / c;  // balanced: every split gets floor/ceil(n/k) pages
            ns[static_cast<size_t>(r)] = k;
            const int chunk = (n + k - 1) / k;
            max_item = std::max(max_item, chunk);
            total += static_cast<double>(n_kv) * (n + k * item_overhead + (k > 1 ? merge_cost : 0.0));
        }
        if (max_item > kMaxItemPages) continue;
        const double est = total / num_workers + 0.5 * (max_item + item_overhead);
        if (best < 0 || est < best - 1e-9) {
            best = est;
            best_ns = ns;
        }
    }

    // Split boundaries per request: the head in best_ns[r]-sized near-equal spans, the
    // last kTailPct% of the pages of every multi-split request in quarter-size spans,
    // so the longest-first dynamic schedule ends on small items and the warps finish
    // together (B200, C2 bench step: warp idle 10.1% -> 4.2% of the launch, +2.3%
    // tokens/s; profiles/ab_r01f_plan_tail.txt).  ASV_PLAN_TAIL=<percent> overrides
    // (tuning only; 0 = equal spans).
    // MHA only: on GQA the extra splits cost more in the merge (one row per query head) than the
    // tail saves (C4 13B GQA-8 engine step: 11 240 -> 10 972 tokens/s with the tail; C1 MHA:
    // 10 600 -> 11 020).
    constexpr int kTailPct = 25;
    static const int tail_env = [] {
        const char* e = getenv("ASV_PLAN_TAIL");
        return e != nullptr ? atoi(e) : -1;
    }();
    const int tail_pct = tail_env >= 0 ? tail_env : (shape->num_q_heads == shape->num_kv_heads ? kTailPct : 0);
    std::vector<std::vector<int32_t>> bounds(static_cast<size_t>(batch));
    for (int r = 0; r < batch; ++r) {
        const int n = npages[static_cast<size_t>(r)], k = best_ns[static_cast<size_t>(r)];
        auto& b = bounds[static_cast<size_t>(r)];
        const int c = (n + k - 1) / k;
        const int tail = k >= 2 ? n * tail_pct / 100 : 0;
        const int small = std::max(2, c / 4);
        if (tail >= 2 * small) {
            const int head = n - tail;
            const int k1 = std::max(1, (head + c - 1) / c);
            for (int s2 = 0; s2 < k1; ++s2) b.push_back(s2 * head / k1);
            const int k2 = tail / small;
            for (int s2 = 0; s2 < k2; ++s2) b.push_back(head + s2 * tail / k2);
        } else {
            for (int s2 = 0; s2 < k; ++s2) b.push_back(s2 * n / k);
        }
        b.push_back(n);
        best_ns[static_cast<size_t>(r)] = static_cast<int32_t>(b.size() - 1);
    }
    int64_t total_splits = 0;
    for (int32_t v : best_ns) total_splits += v;
    const int64_t P = page_indptr[batch];
    const int64_t off_desc = 0;
    int32_t n_merge = 0;
    for (int32_t v : best_ns) n_merge += v > 1 ? 1 : 0;
    const int64_t off_split = off_desc + total_splits * kDescWords;
    const int64_t off_merge = off_split + batch + 1;
    const int64_t need = off_merge + n_merge;
    if (need > plan_cap) return fail(ASV_ERR_INVALID, "plan buffer too small: need " + std::to_string(need));

    asv_attn_plan pl{};
    pl.batch = batch;
    pl.total_splits = static_cast<int32_t>(total_splits);
    pl.num_items = static_cast<int32_t>(total_splits * n_kv);
    pl.num_pages = static_cast<int32_t>(P);
    pl.num_workers = num_workers;
    pl.off_desc = static_cast<int32_t>(off_desc);
    pl.off_split_base = static_cast<int32_t>(off_split);
    pl.off_merge = static_cast<int32_t>(off_merge);
    pl.n_merge = n_merge;
    pl.total_int32 = static_cast<int32_t>(need);
    for (int r = 0, k = 0; r < batch; ++r) {
        if (best_ns[static_cast<size_t>(r)] > 1) plan_buf[off_merge + k++] = r;
    }
    pl.max_item_pages = 0;
    pl.append_missing = 0;

    // split_base: partial slots are request-major (the merge walks them)
    int32_t* sb = plan_buf + off_split;
    sb[0] = 0;
    for (int r = 0; r < batch; ++r) sb[r + 1] = sb[r] + best_ns[static_cast<size_t>(r)];
    // descriptors, counting-sorted by item size descending (stable: request, split)
    std::vector<int32_t> bucket(kMaxItemPages + 2, 0);
    const auto span_of = [&bounds](int r, int s) {
        const auto& b = bounds[static_cast<size_t>(r)];
        return std::pair<int, int>{b[static_cast<size_t>(s)], b[static_cast<size_t>(s) + 1]};
    };
    for (int r = 0; r < batch; ++r) {
        const int k = best_ns[static_cast<size_t>(r)];
        for (int s = 0; s < k; ++s) {
            const auto [pb, pe] = span_of(r, s);
            bucket[static_cast<size_t>(pe - pb)]++;
        }
    }
    std::vector<int64_t> pos(kMaxItemPages + 2, 0);
    for (int sz = kMaxItemPages, acc = 0; sz >= 1; --sz) {
        pos[static_cast<size_t>(sz)] = acc;
        acc += bucket[static_cast<size_t>(sz)];
    }
    for (int r = 0; r < batch; ++r) {
        const int k = best_ns[static_cast<size_t>(r)];
        const int32_t* pages = page_indices + page_indptr[r];
        const int32_t owned = page_indptr[r + 1] - page_indptr[r];
        const int app = seq_lens[r] / 16;
        for (int s = 0; s < k; ++s) {
            const auto [pb, pe] = span_of(r, s);
            int32_t* d = plan_buf + off_desc + pos[static_cast<size_t>(pe - pb)]++ * kDescWords;
            d[0] = r;
            d[1] = sb[r] + s;
            d[2] = pb;
            d[3] = pe;
            d[4] = seq_lens[r];
            d[5] = k;
            d[6] = (s == k - 1 && app < owned) ? pages[app] : -1;
            if (s == k - 1 && app >= owned) ++pl.append_missing;
            d[7] = 0;
            for (int j = 0; j < kMaxItemPages; ++j) d[8 + j] = (pb + j < pe) ? pages[pb + j] : 0;
            pl.max_item_pages = std::max(pl.max_item_pages, pe - pb);
        }
    }
    *plan_out = pl;
    return ASV_OK;
}

size_t asv_attn_workspace_bytes(const asv_attn_shape* shape, int32_t max_batch, int32_t max_total_splits) {
    if (check_shape(shape) != ASV_OK) return 0;
    (void)max_batch;
    const int64_t per = static_cast<int64_t>(shape->num_q_heads) * (128 * 4 + 8);
    // two partial areas (launch_index parity): a launch may leave its partials for the next one
    return static_cast<size_t>(kHeadBytes + 2 * per * std::max<int64_t>(1, max_total_splits));
}

int asv_attn_workspace_init(void* workspace, size_t bytes, void* stream) {
    if (workspace == nullptr || bytes < static_cast<size_t>(kHeadBytes))
        return fail(ASV_ERR_INVALID, "workspace too small");
    cudaError_t e = cudaMemsetAsync(workspace, 0, kHeadBytes, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(workspace)");
    return ASV_OK;
}

int asv_plan_upload(const int32_t* host_plan, int32_t* plan_dev, int64_t n_int32, void* stream) {
    if (host_plan == nullptr || plan_dev == nullptr || n_int32 < 0) return fail(ASV_ERR_INVALID, "bad plan upload");
    if ((reinterpret_cast<uintptr_t>(host_plan) | reinterpret_cast<uintptr_t>(plan_dev)) & 15u)
        return fail(ASV_ERR_INVALID, "plan buffers must be 16-byte aligned");
    cudaError_t e = sm_copy(host_plan, plan_dev, n_int32, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "plan upload");
    return ASV_OK;
}

int asv_decode_attention(const asv_attn_shape* shape, const asv_attn_args* a, void* stream) {
    if (int rc = check_shape(shape)) return rc;
    if (a == nullptr || a->plan == nullptr || a->plan_dev == nullptr)
        return fail(ASV_ERR_INVALID, "null attention args/plan");
    const asv_attn_plan& pl = *a->plan;
    if (pl.batch < 1) return fail(ASV_ERR_INVALID, "empty batch");
    if (a->layer < 0 || a->layer >= shape->num_layers) return fail(ASV_ERR_INVALID, "layer out of range");
    if (a->q == nullptr || a->kv_pool == nullptr || a->out == nullptr)
        return fail(ASV_ERR_INVALID, "null q/kv_pool/out");
    if ((a->k_new == nullptr) != (a->v_new == nullptr))
        return fail(ASV_ERR_INVALID, "k_new and v_new must both be set or both be null");
    const int n_kv = shape->num_kv_heads, n_q = shape->num_q_heads;
    if (a->k_new != nullptr && pl.append_missing > 0)
        return fail(ASV_ERR_INVALID, "KV append requested but " + std::to_string(pl.append_missing) +
                                         " request(s) own no page for position seq_len");
    const bool two_areas = a->defer_merge != 0 || a->prev_out != nullptr;
    const int64_t area = static_cast<int64_t>(pl.total_splits) * n_q * (128 * 4 + 8);
    const int64_t need = kHeadBytes + (two_areas ? 2 : 1) * area;
    if (a->workspace == nullptr || static_cast<int64_t>(a->workspace_bytes) < need)
        return fail(ASV_ERR_INVALID, "workspace too small for plan: need " + std::to_string(need));
    if (a->kv_dtype != ASV_KV_BF16 && a->kv_dtype != ASV_KV_F16)
        return fail(ASV_ERR_INVALID, "kv_dtype must be ASV_KV_BF16 or ASV_KV_F16");
    const bool f16 = a->kv_dtype == ASV_KV_F16;
    const int nw = attn_warps_per_cta(n_q / n_kv, f16);
    if (pl.num_workers < nw || pl.num_workers % nw != 0)
        return fail(ASV_ERR_INVALID, "plan num_workers must be a multiple of the CTA warp count");

    AttnLaunch L{};
    L.group = n_q / n_kv;
    L.grid = pl.num_workers / nw;
    {
        // persistent grid: never more CTAs than can be co-resident (the plan may come from another device)
        int dev = 0;
        cudaGetDevice(&dev);
        int32_t resident = 0;
        if (int rc = asv_attn_num_workers(shape, dev, &resident)) return rc;
        L.grid = std::max(1, std::min(L.grid, resident / nw));
    }
    L.q = a->q;
    L.pool = a->kv_pool;
    if (a->pool_pages < 1) return fail(ASV_ERR_INVALID, "pool_pages must be >= 1 (layer stride of the pool)");
    // layer-major pool (in page groups): consecutive pages of one layer are one slice apart
    L.page_bytes = static_cast<int64_t>(2) * n_kv * kBlockBytes;
    const int64_t gp = pool_group_pages(L.page_bytes, a->pool_pages);
    L.group_pages = static_cast<int32_t>(gp);
    L.group_skip = static_cast<int32_t>(gp * (shape->num_layers - 1));
    L.usable_pages = static_cast<int32_t>(pool_usable_pages(L.page_bytes, a->pool_pages));
    L.layer_off = static_cast<int64_t>(a->layer) * gp * L.page_bytes;
    L.v_off = static_cast<int64_t>(n_kv) * kBlockBytes;
    L.gdesc = a->plan_dev + pl.off_desc;
    L.split_base = a->plan_dev + pl.off_split_base;
    L.pdl = a->pdl != 0;
    L.f16 = f16;
    L.merge_reqs = a->plan_dev + pl.off_merge;
    L.n_merge = pl.n_merge;
    {
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        L.sms = sms > 0 ? sms : 148;
    }
    L.num_items = pl.num_items;
    L.n_kv = n_kv;
    L.n_q = n_q;
    L.k_new = a->k_new;
    L.v_new = a->v_new;
    L.out = a->out;
    L.lse = a->lse;
    char* ws = static_cast<char*>(a->workspace);
    L.work = reinterpret_cast<uint32_t*>(ws) + 4 * (a->launch_index & 1u);
    // partial outputs first (16-byte aligned float4 rows), then the (m, l) pairs; with deferred merges
    // the launch_index parity picks one of two areas (the previous launch's partials are the other)
    const auto area_at = [&](uint32_t parity, float** po, float** pml) {
        char* base = ws + kHeadBytes + (two_areas ? static_cast<int64_t>(parity) * area : 0);
        *po = reinterpret_cast<float*>(base);
        *pml = reinterpret_cast<float*>(base + static_cast<int64_t>(pl.total_splits) * n_q * 512);
    };
    area_at(a->launch_index & 1u, &L.part_o, &L.part_ml);
    L.defer_merge = a->defer_merge != 0;
    L.warm_items = a->l2_warm_items;
    L.warm_pages = a->l2_warm_pages;
    if (a->prev_out != nullptr) {
        float *po = nullptr, *pml = nullptr;
        area_at((a->launch_index - 1u) & 1u, &po, &pml);
        L.prev_part_o = po;
        L.prev_part_ml = pml;
        L.prev_out = a->prev_out;
        L.prev_lse = a->prev_lse;
    }
    L.sm_scale = a->sm_scale;
    L.warp_ts = reinterpret_cast<unsigned long long*>(a->warp_timestamps);
    cudaError_t e = attn_launch(L, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "decode attention launch");
    return ASV_OK;
}

}  // extern "C"
