// C ABI of the decode-attention operator: split-KV planning (K4, host) and the
// K1/K2/K3 launch.  See include/asv.h for the contract and the reference
// functions each entry point replaces.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/asv.h"
#include "asv_internal.h"

namespace asv {

namespace {
thread_local std::string g_last_error;
constexpr int64_t kSemBytes = 256 * 1024;  // 65536 (request, kv head) semaphores
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

// Simulated makespan (page units) of the static round-robin item schedule.
double makespan(const std::vector<int32_t>& npages, const std::vector<int32_t>& ns, int n_kv,
                int workers, double overhead, std::vector<double>& load) {
    load.assign(static_cast<size_t>(workers), 0.0);
    int64_t k = 0;
    double worst = 0.0;
    for (size_t r = 0; r < npages.size(); ++r) {
        const int n = npages[r];
        const int chunk = (n + ns[r] - 1) / ns[r];
        for (int s = 0; s < ns[r]; ++s) {
            const int pages = std::min(n, (s + 1) * chunk) - s * chunk;
            const double cost = pages + overhead + (ns[r] > 1 ? 0.25 : 0.0);
            for (int h = 0; h < n_kv; ++h, ++k) {
                double& w = load[static_cast<size_t>(k % workers)];
                w += cost;
                worst = std::max(worst, w);
            }
        }
    }
    return worst;
}

// Split count so that ceil(n / ceil(n / ns)) == ns: every split non-empty.
int normalize_splits(int n, int ns) {
    ns = std::max(1, std::min(ns, n));
    for (;;) {
        const int chunk = (n + ns - 1) / ns;
        const int ns2 = (n + chunk - 1) / chunk;
        if (ns2 == ns) return ns;
        ns = ns2;
    }
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
int asv_abi_version(void) { return 1; }
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
    *workers_out = sms * blocks * attn_warps_per_cta();
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
    int64_t total_pages = 0;
    int32_t max_pages = 0;
    for (int r = 0; r < batch; ++r) {
        const int32_t s = seq_lens[r];
        if (s < 1) return fail(ASV_ERR_INVALID, "prefix lengths must be >= 1");
        const int32_t np = (s + 15) / 16;
        if (page_indptr[r + 1] - page_indptr[r] < np)
            return fail(ASV_ERR_INVALID, "page table shorter than ceil(seq_len/16) for request " +
                                             std::to_string(r));
        npages[static_cast<size_t>(r)] = np;
        total_pages += np;
        max_pages = std::max(max_pages, np);
    }
    if (page_indptr[0] != 0) return fail(ASV_ERR_INVALID, "page_indptr[0] must be 0");

    // choose per-request split counts: candidates at 1..8 waves of items plus "no split"
    const double overhead = 1.5;  // per item: q load, state reset, epilogue (page units)
    std::vector<int32_t> best_ns(static_cast<size_t>(batch), 1), ns(static_cast<size_t>(batch));
    std::vector<double> load;
    double best = makespan(npages, best_ns, n_kv, num_workers, overhead, load);
    int64_t best_items = static_cast<int64_t>(batch) * n_kv;
    for (int waves = 1; waves <= 8; ++waves) {
        const double target_items = static_cast<double>(waves) * num_workers;
        const double chunk = std::max(2.0, std::ceil(static_cast<double>(total_pages) * n_kv / target_items));
        int64_t items = 0;
        for (int r = 0; r < batch; ++r) {
            const int n = npages[static_cast<size_t>(r)];
            ns[static_cast<size_t>(r)] = normalize_splits(n, static_cast<int>(std::ceil(n / chunk)));
            items += static_cast<int64_t>(ns[static_cast<size_t>(r)]) * n_kv;
        }
        const double ms = makespan(npages, ns, n_kv, num_workers, overhead, load);
        if (ms < best - 1e-9 || (std::fabs(ms - best) <= 1e-9 && items < best_items)) {
            best = ms;
            best_ns = ns;
            best_items = items;
        }
    }

    int64_t total_splits = 0;
    for (int32_t v : best_ns) total_splits += v;
    const int64_t P = page_indptr[batch];
    // item_tab holds int2 pairs: keep it 8-byte aligned inside the int32 buffer
    const int64_t off_tab = (batch + (batch + 1) + P + (batch + 1) + 1) & ~int64_t{1};
    const int64_t need = off_tab + 2 * total_splits;
    if (need > plan_cap) return fail(ASV_ERR_INVALID, "plan buffer too small: need " + std::to_string(need));

    asv_attn_plan pl{};
    pl.batch = batch;
    pl.total_splits = static_cast<int32_t>(total_splits);
    pl.num_items = static_cast<int32_t>(total_splits * n_kv);
    pl.num_pages = static_cast<int32_t>(P);
    pl.num_workers = num_workers;
    pl.off_seq_lens = 0;
    pl.off_page_indptr = batch;
    pl.off_page_indices = pl.off_page_indptr + batch + 1;
    pl.off_split_indptr = static_cast<int32_t>(pl.off_page_indices + P);
    pl.off_item_tab = static_cast<int32_t>(off_tab);
    pl.total_int32 = static_cast<int32_t>(need);
    pl.max_item_pages = 0;

    std::memcpy(plan_buf + pl.off_seq_lens, seq_lens, sizeof(int32_t) * batch);
    std::memcpy(plan_buf + pl.off_page_indptr, page_indptr, sizeof(int32_t) * (batch + 1));
    std::memcpy(plan_buf + pl.off_page_indices, page_indices, sizeof(int32_t) * P);
    int32_t* sp = plan_buf + pl.off_split_indptr;
    int32_t* tab = plan_buf + pl.off_item_tab;
    sp[0] = 0;
    int64_t g = 0;
    for (int r = 0; r < batch; ++r) {
        const int n = npages[static_cast<size_t>(r)];
        const int k = best_ns[static_cast<size_t>(r)];
        const int chunk = (n + k - 1) / k;
        pl.max_item_pages = std::max(pl.max_item_pages, chunk);
        for (int s = 0; s < k; ++s, ++g) {
            tab[2 * g] = r;
            tab[2 * g + 1] = s;
        }
        sp[r + 1] = static_cast<int32_t>(g);
    }
    *plan_out = pl;
    return ASV_OK;
}

size_t asv_attn_workspace_bytes(const asv_attn_shape* shape, int32_t max_batch, int32_t max_total_splits) {
    if (check_shape(shape) != ASV_OK) return 0;
    (void)max_batch;
    const int64_t per = static_cast<int64_t>(shape->num_q_heads) * (128 * 4 + 8);
    return static_cast<size_t>(kSemBytes + per * std::max<int64_t>(1, max_total_splits));
}

int asv_attn_workspace_init(void* workspace, size_t bytes, void* stream) {
    if (workspace == nullptr || bytes < static_cast<size_t>(kSemBytes))
        return fail(ASV_ERR_INVALID, "workspace too small");
    cudaError_t e = cudaMemsetAsync(workspace, 0, kSemBytes, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync(workspace)");
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
    if (static_cast<int64_t>(pl.batch) * n_kv * 4 > kSemBytes)
        return fail(ASV_ERR_INVALID, "batch * num_kv_heads exceeds the semaphore capacity");
    const int64_t need = kSemBytes + static_cast<int64_t>(pl.total_splits) * n_q * (128 * 4 + 8);
    if (a->workspace == nullptr || static_cast<int64_t>(a->workspace_bytes) < need)
        return fail(ASV_ERR_INVALID, "workspace too small for plan: need " + std::to_string(need));
    const int nw = attn_warps_per_cta();
    if (pl.num_workers < nw || pl.num_workers % nw != 0)
        return fail(ASV_ERR_INVALID, "plan num_workers must be a multiple of the CTA warp count");

    AttnLaunch L{};
    L.group = n_q / n_kv;
    L.grid = pl.num_workers / nw;
    L.q = a->q;
    L.pool = a->kv_pool;
    L.page_bytes = static_cast<int64_t>(shape->num_layers) * 2 * n_kv * kBlockBytes;
    L.layer_off = static_cast<int64_t>(a->layer) * 2 * n_kv * kBlockBytes;
    L.v_off = static_cast<int64_t>(n_kv) * kBlockBytes;
    L.seq_lens = a->plan_dev + pl.off_seq_lens;
    L.page_indptr = a->plan_dev + pl.off_page_indptr;
    L.page_indices = a->plan_dev + pl.off_page_indices;
    L.split_indptr = a->plan_dev + pl.off_split_indptr;
    L.item_tab = a->plan_dev + pl.off_item_tab;
    L.num_items = pl.num_items;
    L.n_kv = n_kv;
    L.n_q = n_q;
    L.k_new = a->k_new;
    L.v_new = a->v_new;
    L.out = a->out;
    L.lse = a->lse;
    char* ws = static_cast<char*>(a->workspace);
    L.sem = reinterpret_cast<int32_t*>(ws);
    // partial outputs first (16-byte aligned float4 rows), then the (m, l) pairs
    L.part_o = reinterpret_cast<float*>(ws + kSemBytes);
    L.part_ml = reinterpret_cast<float*>(ws + kSemBytes + static_cast<int64_t>(pl.total_splits) * n_q * 512);
    L.sm_scale = a->sm_scale;
    cudaError_t e = attn_launch(L, static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) return cuda_fail(e, "decode attention launch");
    return ASV_OK;
}

}  // extern "C"
